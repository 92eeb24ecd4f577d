# compute-sanitizer records for the hot kernels (profiles/r2/sanitizer_*.txt)
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san/$tool.txt
done
