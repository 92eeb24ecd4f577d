"""Text summary of an ncu capture exported by scripts/gpu_ncu2.sh (raw page
CSV + SASS source CSV): key counters, FP64 pipe budget, phase breakdown.
usage: python scripts/ncu_text.py raw_TAG.csv sass_TAG.csv.gz > profiles/rN/ncu_x.txt"""
import csv, subprocess, sys
from pathlib import Path

raw_path, sass_path = sys.argv[1], sys.argv[2]
raw = list(csv.reader(open(raw_path)))
d = dict(zip(raw[0], raw[2]))
u = dict(zip(raw[0], raw[1]))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
print(f"# ncu --set full --clock-control none (one launch); source: {Path(raw_path).name}")
for k in keys:
    if k in d:
        print(f"{k:78s} {d[k]} {u.get(k, '')}")
here = Path(__file__).resolve().parent
print("\n## FP64 pipe budget (scripts/ncu_pipe.py)")
print(subprocess.run([sys.executable, str(here / "ncu_pipe.py"), sass_path, raw_path], capture_output=True,
                     text=True).stdout)
print("## phase breakdown: SASS split at barriers (scripts/ncu_regions.py)")
print(subprocess.run([sys.executable, str(here / "ncu_regions.py"), sass_path], capture_output=True,
                     text=True).stdout)
