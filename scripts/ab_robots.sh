#!/bin/bash
# Dev A/B of the robots-on-device call (fsg_batch_step_dynamic, bench's robot
# leg on c5): each variant copied over the in-tree library in turn.
libs=$1; out=gpurun_out/rod.txt
cp paper_2206_01683_b200/libfsg.so /tmp/libfsg_orig.so
for r in 1 2; do for l in $libs; do
  cp paper_2206_01683_b200/ab/$l.so paper_2206_01683_b200/libfsg.so
  python bench.py --workload c5 --steps 50 --warmup 5 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['e2e_robots_on_device']; print('$l', r['value'], r['call_us'])" >> $out
done; done
cp /tmp/libfsg_orig.so paper_2206_01683_b200/libfsg.so
