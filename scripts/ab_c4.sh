#!/bin/bash
# Dev A/B of library variants on the 512^3 pure-fluid K4 (c4) and c3: bench lines interleaved.
libs=$1; out=gpurun_out/ab_c4.txt
for r in 1 2; do for l in $libs; do
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c4 --steps 20 --warmup 3 \
    --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $l', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $out
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload c3 --steps 300 --warmup 10 \
    --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $l', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fluid_only'])" >> $out
done; done
