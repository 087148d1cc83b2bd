#!/bin/bash
# Dev A/B of environment switches on the same library: bench lines for each
# "NAME=VAL ..." setting, interleaved, two rounds.
#   scripts/ab_env.sh "FSG_KM_CHAIN=0|FSG_KM_CHAIN=1" "c2 c3"
IFS='|' read -ra sets <<< "$1"; wls=${2:-"c2 c3"}; out=gpurun_out/ab_env.txt
for r in 1 2; do for w in $wls; do for e in "${sets[@]}"; do
  env $e python bench.py --workload $w --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w [$e]', d['value'], d['ms_per_step'], d['roofline']['frac'], (d['roofline'].get('fluid_only') or {}).get('ms'), d['e2e']['value'])" >> $out
done; done; done
