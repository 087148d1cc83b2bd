out=gpurun_out/kmsm.txt; rm -f $out
for r in 1 2; do for w in c3 c2; do for tl in 0 1; do for k in 0 2.5 3 4; do
  FSG_TILE_LIST=$tl FSG_KM_PER_SM=$k python bench.py --workload $w --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w tl=$tl km=$k', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done; done; done
sort $out
