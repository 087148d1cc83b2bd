out=gpurun_out/pad.txt; rm -f $out
for r in 1 2; do for p in 0 32 128 1056 4160; do
  FSG_PLANE_PAD=$p python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 pad $p', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
for p in 0 32 1056; do
  FSG_PLANE_PAD=$p python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 pad $p', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fluid_only']['ms'])" >> $out
done
FSG_PLANE_PAD=32 python -m pytest tests/test_parity_gpu.py tests/test_slab_gpu.py -q 2>&1 | tail -2 >> $out
cat $out
