out=gpurun_out/np.txt; rm -f $out
for r in 1 2; do for cfg in "base3:0" "np2m5:0" "np4m4:4" "np4m5:4"; do l=${cfg%%:*}; z=${cfg##*:};
  FSG_K4_ZC=$z FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c3 --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $l zc=$z', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
done; done
sort $out
