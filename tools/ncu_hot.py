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
