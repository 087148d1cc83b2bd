#!/bin/bash
# Dev A/B of library variants on the batched c5 round (and c1 / c2 sanity).
libs=$1; out=gpurun_out/ab_c5.txt
for r in 1 2; do for l in $libs; do
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c5 --steps 300 --warmup 10 \
    --e2e-steps 10 --no-cpu-baseline --no-robot-leg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $l', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c1 --steps 300 --warmup 10 \
    --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $l', d['value'], d['ms_per_step'], d['roofline']['frac'], (d['roofline'].get('fluid_only') or {}).get('ms'))" >> $out
done; done
