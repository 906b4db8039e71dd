"""Summarise an ncu --set full capture into profiles/ncu_summary.json (dev aid).

Usage: python tools/ncu_summarize.py REPORT.ncu-rep KEY KERNEL_REGEX UNITS_PER_LAUNCH SOURCE
Reads `ncu -i REPORT --page raw --csv`, averages the launches whose name
matches KERNEL_REGEX, and stores DRAM bytes per launch (read + write), the
duration and the key cache rates under KEY.  bench.py reads
dram_bytes_per_launch as roofline.traffic.
"""
import csv, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
        "msecond": 1e3, "%": 1, "sector": 1, "": 1}


def main():
    rep, key, rx, units, source = sys.argv[1:6]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units_row, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")

    def col(name, row):
        i = hdr.index(name)
        return float(row[i].replace(",", "")) * UNIT.get(units_row[i], 1)

    sel = [r for r in data if re.search(rx, r[ki])]
    if not sel:
        sys.exit(f"no launch matches {rx}")
    avg = lambda name: sum(col(name, r) for r in sel) / len(sel)
    s = {
        "dram_bytes_per_launch": avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum"),
        "dram_read_bytes": avg("dram__bytes_read.sum"),
        "dram_write_bytes": avg("dram__bytes_write.sum"),
        "duration_us": avg("gpu__time_duration.sum"),
        "units_per_launch": int(float(units)),
        "dram_throughput_pct": avg("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": avg("lts__t_sector_hit_rate.pct"),
        "l1_hit_pct": avg("l1tex__t_sector_hit_rate.pct"),
        "achieved_occupancy_pct": avg("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "l1_tag_sectors_per_launch": (avg("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
                                      + avg("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum")),
        "l2_requests_per_launch": avg("lts__t_requests_srcunit_tex.sum"),
        "l1_to_l2_req_active_pct": avg(
            "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "launches_averaged": len(sel),
        "source": source,
    }
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allv = json.load(open(path)) if os.path.exists(path) else {}
    allv[key] = s
    json.dump(allv, open(path, "w"), indent=1)
    print(json.dumps({key: s}, indent=1))


if __name__ == "__main__":
    main()
