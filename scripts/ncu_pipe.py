"""FP64 pipe budget of a kernel from an ncu SASS export: DMMA.8x8x4 = 16 SMSP
cycles (256 FMA at 16 FMA/clk/SMSP), D* SIMT warp-instruction = 2 cycles,
MUFU.*64* = ? (counted separately). usage: python scripts/ncu_pipe.py sass.csv.gz raw.csv"""
import csv, gzip, io, sys, collections
rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), encoding="utf-8")))
hdr = rows[1]; ix = {k: i for i, k in enumerate(hdr)}
cnt = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) - 5: continue
    src = r[ix["Source"]].strip().split()
    if not src: continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    cnt[op.split(".")[0] if not op.startswith("DMMA") else op] += float(r[ix["Instructions Executed"]] or 0)
raw = list(csv.reader(open(sys.argv[2])))
d = dict(zip(raw[0], raw[2]))
dur = float(d["gpu__time_duration.sum"].replace(",", ""))  # ns or us per unit row
unit = raw[1][raw[0].index("gpu__time_duration.sum")]
dur_s = dur * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
               "s": 1.0}.get(unit, 1e-9)
clk = float(d.get("smsp__cycles_elapsed.avg.per_second", "0").replace(",", "") or 0)
nsm = 148
dmma = sum(v for k, v in cnt.items() if k.startswith("DMMA"))
dsimt = sum(cnt[k] for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET"))
mufu = cnt["MUFU"]
cyc_dmma = dmma * 16
cyc_simt = dsimt * 2
smsp_cycles_avail = dur_s * 1.965e9 * nsm * 4
print(f"duration {dur_s*1e3:.2f} ms; DMMA.8x8x4 {dmma:.4g}  DP-SIMT {dsimt:.4g}  MUFU {mufu:.3g}")
print(f"pipe cycles: DMMA {cyc_dmma:.4g} ({100*cyc_dmma/smsp_cycles_avail:.1f}% of SMSP-cycles)  SIMT {cyc_simt:.4g} "
      f"({100*cyc_simt/smsp_cycles_avail:.1f}%)  total {100*(cyc_dmma+cyc_simt)/smsp_cycles_avail:.1f}%")
print("top DP:", {k: f"{cnt[k]:.3g}" for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "MUFU", "FSEL", "F2F")})
