out=gpurun_out/fpair.txt; rm -f $out
for r in 1 2; do for l in base2 fpair; do for z in 0 2; do
  FSG_K4F_ZC=$z FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $l zc=$z', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done;
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $l', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fluid_only']['ms'])" >> $out
done; done
sort $out
