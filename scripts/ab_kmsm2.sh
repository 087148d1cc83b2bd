out=gpurun_out/kmsm2.txt; rm -f $out
timeout 600 python -m pytest tests/test_skin_gpu.py tests/test_ref_robot_gpu.py tests/test_batch_gpu.py tests/test_nonfinite_gpu.py -q 2>&1 | tail -1 >> $out
for r in 1 2; do for k in 1.5 2 3 4; do
  FSG_KM_PER_SM=$k python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 km=$k', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
sort $out
