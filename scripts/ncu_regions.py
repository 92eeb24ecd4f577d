"""Phase-level attribution of an ncu SASS source export (no GPU needed):
split the kernel's SASS at barrier opcodes and sum stall samples, executed
instructions and stall reasons per region.
usage: python scripts/ncu_regions.py sass_TAG.csv.gz"""
import csv, gzip, io, sys, collections

path = sys.argv[1]
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), encoding="utf-8")))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
split_ops = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else {"BAR", "WARPSYNC"}
regions = []
def new(name):
    return {"name": name, "samples": 0.0, "exec": 0.0, "ops": collections.Counter(), "stall": collections.Counter(),
            "dp": 0.0, "dmma": 0.0, "n": 0}
cur = new("start")
for r in rows[2:]:
    if len(r) < len(hdr) - 5:
        continue
    src = r[ix["Source"]].strip()
    parts = src.split()
    op = parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "?")
    opb = op.split(".")[0]
    if opb in split_ops:
        regions.append(cur)
        cur = new(f"{r[ix['Address']][-5:]} {op}")
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = float(r[ix["Instructions Executed"]] or 0)
    cur["samples"] += s
    cur["exec"] += ex
    cur["n"] += 1
    cur["ops"][opb] += ex
    if opb in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
        cur["dp"] += ex
    if opb == "DMMA":
        cur["dmma"] += ex
    for k in stall_cols:
        cur["stall"][k[6:]] += float(r[ix[k]] or 0)
regions.append(cur)
tot = sum(x["samples"] for x in regions) or 1
totex = sum(x["exec"] for x in regions) or 1
print(f"total samples {tot:.0f}, executed warp-instructions {totex:.4g}")
for x in regions:
    if x["samples"] / tot < 0.005 and x["exec"] / totex < 0.005:
        continue
    top = ", ".join(f"{k} {100*v/max(x['samples'],1):.0f}%" for k, v in x["stall"].most_common(4))
    ops = ", ".join(f"{k}:{v:.3g}" for k, v in x["ops"].most_common(6))
    print(f"[{x['name']:>22s}] n={x['n']:4d} samples {100*x['samples']/tot:5.1f}%  exec {100*x['exec']/totex:5.1f}%  "
          f"DMMA {x['dmma']:.3g} DP {x['dp']:.3g}\n      stalls: {top}\n      ops: {ops}")
