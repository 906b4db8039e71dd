"""Sum DRAM bytes of the second tv_bridges call in gpurun_out/br_dram.csv into
profiles/ncu_summary.json (bridges_D) -- bench.py reports it as roofline.traffic."""
import collections, csv, json, os, re, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "br_dram.csv")
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                            "Metric Unit", "ID"))
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
      "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * SC.get(r[ui], 1)
L = list(launch.values())
starts = [i for i, d in enumerate(L) if "k_iota" in d["name"]]
second = L[starts[1]:] if len(starts) > 1 else L
sel = [d for d in second if re.search(r"(^|\s|::|>::)k_", d["name"])]
tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in sel)
dur = sum(d.get("gpu__time_duration.sum", 0) for d in sel)
p = os.path.join(ROOT, "profiles", "ncu_summary.json")
s = json.load(open(p))
s["bridges_D"] = {"dram_bytes_per_call": tot, "kernels_per_call": len(sel),
                  "sum_kernel_us_cold": dur, "n": 32022410, "m": 256000000,
                  "model_bytes": 41 * 256000000 + 108 * 32022410,
                  "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                            "gpu__time_duration.sum over every kernel of the second tv_bridges "
                            "call on config D (tools/gpu_br_dram.sh, tools/br_dram_summary.py)"}
json.dump(s, open(p, "w"), indent=1)
print(json.dumps(s["bridges_D"], indent=1))
top = sorted(sel, key=lambda d: -(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)))
for d in top[:10]:
    print(re.sub(r"\(.*", "", d["name"])[:50],
          round((d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e9, 3), "GB",
          round(d["gpu__time_duration.sum"], 1), "us")
