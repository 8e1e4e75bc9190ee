"""Top SASS lines by warp-stall samples for each kernel of an ncu report (source page)."""
import csv
import subprocess
import sys

rep, ntop = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        kern.append(cur)
    elif r and r[0] == "Address" and cur:
        cur[1] = r
    elif cur and cur[1] and len(r) == len(cur[1]):
        cur[2].append(r)
for name, hdr, data in kern:
    i_s, i_src, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
    tot = sum(int(r[i_s]) for r in data) or 1
    print("==", name[:120], "samples", tot)
    for r in sorted(data, key=lambda r: -int(r[i_s]))[:ntop]:
        print(f"{int(r[i_s]) * 100 / tot:5.1f}% {r[0][-5:]} {r[i_ex]:>9} {r[i_src].strip()[:90]}")


def by_line(rep, ntop=30):
    """Stall samples per CUDA source line (cuda,sass view)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg, fname, func = {}, None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Function Name":
            func = r[1][:60]
        elif r[0] not in ("", "Line No") and len(r) > 4 and r[4].isdigit():
            key = (func, fname, int(r[0]))
            agg[key] = (agg.get(key, (0, ""))[0] + int(r[4]), r[1].strip()[:90])
    for func in sorted({k[0] for k in agg}):
        items = [(k, v) for k, v in agg.items() if k[0] == func]
        tot = sum(v[0] for _, v in items) or 1
        print("==", func, "samples", tot)
        for k, v in sorted(items, key=lambda kv: -kv[1][0])[:ntop]:
            print(f"{v[0] * 100 / tot:5.1f}% {k[1]}:{k[2]:<5} {v[1]}")


if len(sys.argv) > 3 and sys.argv[3] == "lines":
    by_line(rep, ntop)
