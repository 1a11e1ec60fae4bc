"""Print per-launch metrics from an ncu --csv launch list. usage: launches.py file [filter]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg.setdefault((d['ID'], d['Kernel Name'][:50]), {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
for (i, n), v in agg.items():
    if flt in n:
        print(i, n, v.get('gpu__time_duration.sum'), round(v.get('dram__bytes_read.sum', 0) / 1e6, 1), round(v.get('dram__bytes_write.sum', 0) / 1e6, 1))
