# round-2 evidence: bench lines (both arms), ncu launch list of the bench command,
# ncu --set full of the dominant kernel (4.09M tets) and of the curved kernel
mkdir -p gpurun_out/r2ev gpurun_out/ncu
( lscpu; nproc; free -g; nvidia-smi ) > gpurun_out/r2ev/box.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2ev/bench.json 2> gpurun_out/r2ev/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2ev/bench_ref.json 2> gpurun_out/r2ev/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2ev/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --curved-n 0 > gpurun_out/r2ev/launches.log 2>&1; echo "launches rc=$?"
bash scripts/gpu_ncu2.sh r2row k_rhs_row "--curved-n 0"
bash scripts/gpu_ncu2.sh r2rowc k_rhs_rowc "--n 8 --curved-n 32"
python - <<'PY'
import csv, json
raw = list(csv.reader(open("gpurun_out/ncu/raw_r2row.csv")))
d = dict(zip(raw[0], raw[2]))
def num(k):
    return float(d[k].replace(",", ""))
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
units = dict(zip(raw[0], raw[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale.get(units["dram__bytes_read.sum"], 1)
wr *= scale.get(units["dram__bytes_write.sum"], 1)
K = 6 * 88 ** 3
B = 160 * 35 + 80 * 64 + 208 + 32
json.dump({"kernel": d.get("Kernel Name"), "workload": "make_cube_mesh(88) = 4,088,832 tets, P=4, one RK stage",
           "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "algorithmic_bytes_per_launch": K * B,
           "source": "profiles/r2/ncu_k_rhs_row.txt (ncu --set full --clock-control none, one launch)"},
          open("gpurun_out/r2ev/ncu_rhs_p4.json", "w"), indent=1)
print("traffic", rd + wr)
PY
timeout 1200 python scripts/bench_configs.py --large-only >> gpurun_out/r2ev/configs_large.jsonl 2> gpurun_out/r2ev/configs_large.err; echo "large rc=$?"
