"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin."""
import re, sys
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = m.group(1)
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in rows.items():
    if flt in k:
        print(f"{k[:60]:60s} regs={v.get('regs')} spill={v.get('spill')}")
