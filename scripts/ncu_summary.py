"""Summarise an ncu report (run here, no GPU): key throughput metrics, stall
reasons, top SASS opcodes by stall samples. usage: python scripts/ncu_summary.py rep [--json out]"""
import collections, csv, io, json, subprocess, sys

rep = sys.argv[1]
def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units, v = raw[0], raw[1], raw[2]
d = dict(zip(h, v)); u = dict(zip(h, units))
def g(k):
    x = d.get(k, "nan").replace(",", "")
    try: return float(x)
    except ValueError: return x
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]
out = {}
for k in keys:
    if k in d:
        out[k] = g(k); print(f"{k:70s} {d[k]} {u.get(k,'')}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) for k, x in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and x.replace('.','').isdigit()}
tot = sum(st.values()) or 1
print("stall reasons:")
out["stalls_pct"] = {}
for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
    print(f"  {k:28s} {100*x/tot:5.1f}%"); out["stalls_pct"][k] = round(100 * x / tot, 1)
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(rows) > 2:
    hdr = rows[1]
    i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed")
    byop = collections.Counter(); exop = collections.Counter(); tot = 0
    for r in rows[2:]:
        if len(r) <= i_s: continue
        s = float(r[i_s] or 0); src = r[i_src].strip(); ex = float(r[i_ex] or 0); tot += s
        parts = src.split(); op = parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "?")
        byop[op.split(".")[0]] += s; exop[op.split(".")[0]] += ex
    print("stall samples by opcode (executed warp-instructions):")
    out["opcodes"] = {}
    for op, s in byop.most_common(16):
        print(f"  {op:10s} {100*s/tot:5.1f}%  {exop[op]:.3g}"); out["opcodes"][op] = [round(100*s/tot,1), exop[op]]
if "--json" in sys.argv:
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
