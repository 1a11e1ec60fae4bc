"""Summarise an ncu launch list (+ a --set full report) into profiles/<tag>_summary.md.
usage: python tools/summarize_profiles.py TAG"""
import collections, csv, io, os, subprocess, sys
tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
out = [f"# ncu summary {tag}\n"]
plain = open(os.path.join(G, f"{tag}_plain.log")).read().strip().splitlines()
out.append("Command: `python bench.py --steps 1 --warmup 3 --iters 5 --no-cpu-baseline --no-gmres --no-pnpn --no-graph` (1 B200); "
           "launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
           "--clock-control none` (cold-cache, serialised: compare shares, not absolutes).\n")
out.append("Plain run JSON line (not under ncu):\n\n```\n" + (plain[-1] if plain else "") + "\n```\n")
rows = list(csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for v in per.values():
    n = v["name"].split("(")[0]
    a = agg[n]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += v.get("dram__bytes_read.sum", 0) / 1e6
    a[3] += v.get("dram__bytes_write.sum", 0) / 1e6
tot = sum(a[1] for a in agg.values())
out.append("| kernel | launches | total us | share | avg us | DRAM read MB/launch | DRAM write MB/launch |\n|---|---|---|---|---|---|---|")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| `{n}` | {a[0]} | {a[1]:.1f} | {100 * a[1] / tot:.1f}% | {a[1] / a[0]:.2f} | {a[2] / a[0]:.1f} | {a[3] / a[0]:.1f} |")
rep = os.path.join(G, f"{tag}_full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u = rr[0], rr[1]
    ix = {k: i for i, k in enumerate(h)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
    out.append("\n## `--set full` captures (ITERS=3 tools/prof_cg.py: the CG kernels on the c2 mesh)\n")
    out.append("| kernel | " + " | ".join(keys) + " |")
    out.append("|---" * (len(keys) + 1) + "|")
    for d in rr[2:]:
        out.append(f"| `{d[ix['Kernel Name']][:40]}` | " + " | ".join(f"{d[ix[k]]} {u[ix[k]]}" if k in ix else "-" for k in keys) + " |")
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
