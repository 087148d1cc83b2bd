out=gpurun_out/tail.txt; rm -f $out
for r in 1 2; do for t in 3 0 1 6; do
  FSG_K4_TAIL=$t python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 tail=$t', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
sort $out
