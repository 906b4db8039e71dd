"""Markdown table of ncu --set full captures (dev aid): one row per launch.

  python tools/ncu_table.py REPORT.ncu-rep [REPORT2 ...]
"""
import csv, io, subprocess, sys

COLS = [("duration", "gpu__time_duration.sum"), ("DRAM read", "dram__bytes_read.sum"),
        ("DRAM write", "dram__bytes_write.sum"),
        ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 hit %", "lts__t_sector_hit_rate.pct"),
        ("L1/TEX %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"),
        ("ld B/sector", "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
        ("st B/sector", "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio")]


def short(name):
    name = name.split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.replace("void ", "").replace("ettg::", "").strip()


def main():
    print("| kernel | " + " | ".join(c for c, _ in COLS) + " |")
    print("|---|" + "---:|" * len(COLS))
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, u = rows[0], rows[1]
        for r in rows[2:]:
            cells = []
            for _, m in COLS:
                if m not in h:
                    cells.append("-")
                    continue
                i = h.index(m)
                v, unit = r[i], u[i]
                try:
                    f = float(v.replace(",", ""))
                    v = f"{f:.3g}"
                except ValueError:
                    pass
                cells.append(f"{v} {unit}".strip() if unit not in ("%", "") else v)
            print(f"| `{short(r[h.index('Kernel Name')])}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
