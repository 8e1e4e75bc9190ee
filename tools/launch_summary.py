"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name):
    m = re.search(r"(ttg::\S*?_kernel)(<[^(]*>)?", name)
    if m:
        tmpl = m.group(2) or ""
        return m.group(1) + tmpl.replace("ttg::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:60]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        k = short(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>9s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {v[0]:8d} {v[1] / 1e3:10.3f} {v[1] / v[0]:9.1f} {100 * v[1] / tot:6.2f}%")
    print(f"{'TOTAL':70s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
