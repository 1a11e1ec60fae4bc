"""Print SASS context around the hottest instructions. usage: rep filter [ctx] [top]"""
import csv, io, subprocess, sys
rep, flt = sys.argv[1], sys.argv[2]
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 8
top = int(sys.argv[4]) if len(sys.argv) > 4 else 3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
for b in out.split('"Kernel Name",')[1:]:
    name = b.split("\n", 1)[0]
    if flt not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]; i_src = h.index("Source"); i_s = h.index("Warp Stall Sampling (All Samples)"); i_ex = h.index("Instructions Executed")
    data = [(int(r[i_s] or 0), r[i_src].strip(), r[i_ex]) for r in rows[1:] if len(r) > i_s]
    order = sorted(range(len(data)), key=lambda q: -data[q][0])[:top]
    for q in order:
        print(f"---- around #{q} ({data[q][0]} samples)")
        for z in range(max(0, q - ctx), min(len(data), q + ctx + 1)):
            print(f"{'>>' if z == q else '  '} {data[z][0]:6d} {data[z][2]:>9s}  {data[z][1]}")
    break
