"""Summarise an ncu report's source page: top SASS instructions by warp-stall samples.
usage: python tools/ncu_hot.py report.ncu-rep [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
seen = set()
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if want not in name or name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    i_src, i_s, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = [(int(r[i_s] or 0), r[i_src].strip(), r[i_ex]) for r in rows[1:] if len(r) > i_s]
    tot = sum(d[0] for d in data)
    print(f"== {name}  total samples {tot}, {len(data)} instructions")
    for s, src, ex in sorted(data, reverse=True)[:top]:
        print(f"{100.0*s/max(tot,1):6.2f}%  {s:7d}  exec={ex:>9}  {src}")
