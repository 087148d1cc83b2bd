out=gpurun_out/kmsm3.txt; rm -f $out
for r in 1 2; do for k in 3 4 2.5; do
  FSG_KM_PER_SM=$k python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 km=$k', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
sort $out
