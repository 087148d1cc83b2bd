#!/bin/bash
# Dev A/B: bench lines of several library variants (paper_2206_01683_b200/ab/*.so)
# interleaved, two rounds.  usage: scripts/ab_bench.sh "orig spec pair" "c2 c1 c3"
libs=$1; wls=${2:-"c2 c1 c3"}; out=gpurun_out/ab.txt
for r in 1 2; do for w in $wls; do for l in $libs; do
  FSG_LIB=$PWD/paper_2206_01683_b200/ab/$l.so python bench.py --workload $w --steps 300 --warmup 10 \
    --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $l', d['value'], d['ms_per_step'], d['roofline']['frac'], (d['roofline'].get('fluid_only') or {}).get('ms'))" >> $out
done; done; done
