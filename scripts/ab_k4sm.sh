out=gpurun_out/k4sm.txt; rm -f $out
for r in 1 2; do for p in 6 5 4 3; do
  FSG_K4_PER_SM=$p python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 k4/sm $p', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
cat $out
