"""Summarise an ncu launch list (gpu__time_duration.sum CSV) into a markdown table.

Usage: python tools/launch_share.py launches.csv "command text" > profiles/rNN_launches.md
"""
import collections, csv, re, sys


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("ettg::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.strip()


def main():
    path, cmd = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
        k = short(r[ki])
        a = agg.setdefault(k, [0.0, 0])
        a[0] += float(r[vi].replace(",", "")) * scale
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    print("# Launch list (ncu gpu__time_duration.sum, --clock-control none)\n")
    print(f"Command: `{cmd}` on 1x B200.")
    print("Per-launch times are cold-cache and serialised; compare shares, not absolutes.\n")
    print("| kernel | launches | total us | us/launch | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        if t / tot < 0.001:
            continue
        print(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / tot:.1f}% |")
    print(f"\nTotal {tot:.1f} us over {sum(v[1] for v in agg.values())} launches.")


if __name__ == "__main__":
    main()
