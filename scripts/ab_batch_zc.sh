out=gpurun_out/bzc.txt; rm -f $out
for r in 1 2; do for z in 1 2 4; do
  FSG_BATCH_ZC=$z python bench.py --workload c5 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline --no-robot-leg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 zc $z', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
cat $out
