#!/bin/bash
# Dev A/B of the C++-host e2e step (host_e2e links libfsg.so by rpath): each
# variant is copied over the in-tree library in turn (scratch copy on the box).
libs=$1; wls=${2:-"c3 c2"}; out=gpurun_out/ab_e2e.txt
cp paper_2206_01683_b200/libfsg.so /tmp/libfsg_orig.so
for r in 1 2; do for w in $wls; do for l in $libs; do
  cp paper_2206_01683_b200/ab/$l.so paper_2206_01683_b200/libfsg.so
  python bench.py --workload $w --steps 50 --warmup 5 --e2e-steps 100 --no-cpu-baseline --no-robot-leg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $l', d['ms_per_step'], d['e2e']['value'], d['e2e'].get('us_per_step'))" >> $out
done; done; done
cp /tmp/libfsg_orig.so paper_2206_01683_b200/libfsg.so
