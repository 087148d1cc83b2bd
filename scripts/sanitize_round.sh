set -x
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/san
for tool in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_steps.py 2 > gpurun_out/san/$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log >> gpurun_out/san/summary.txt
done
timeout 600 python -m pytest tests/test_long_parity_gpu.py -k 10k -q > gpurun_out/san/t10k.log 2>&1; tail -3 gpurun_out/san/t10k.log >> gpurun_out/san/summary.txt
cat gpurun_out/san/summary.txt
