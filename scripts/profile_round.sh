#!/bin/bash
# ncu evidence for profiles/ (run on a B200 under gpurun, one GPU).  Every
# command runs once plainly and must exit 0 before it is run under ncu
# (/opt/skills/guides/B200_PROFILING.md).  Outputs in gpurun_out/<tag>_*.
set -u
tag=${1:-r1b}
out=gpurun_out
mkdir -p $out
C2="python bench.py --workload c2 --steps 30 --warmup 5 --e2e-steps 5 --no-cpu-baseline"
C3="python bench.py --workload c3 --steps 12 --warmup 4 --e2e-steps 2 --no-cpu-baseline"
C4="python bench.py --workload c4 --steps 6 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
C5="python bench.py --workload c5 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
# launch lists of the headline workload (c3, bench.py's default) and of c2
# (cold-cache, serialised)
$C3 > $out/${tag}_c3_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/${tag}_c3_launches.csv $C3 > $out/${tag}_c3_ncu_list.log 2>&1
$C2 > $out/${tag}_c2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file $out/${tag}_c2_launches.csv $C2 > $out/${tag}_c2_ncu_list.log 2>&1
# full sections: the coupled pair at c2 (PROFILE_SKIP_C2_FULL=1: skip, keeps
# gpurun_out under the 64 MiB copy-back limit)
[ "${PROFILE_SKIP_C2_FULL:-0}" = 1 ] || ncu --set full --clock-control none --import-source on -k regex:"k_collide_band|k_markers_fix|k_markers_skin" \
    -s 20 -c 4 -o $out/${tag}_c2_full $C2 > $out/${tag}_c2_ncu_full.log 2>&1
# c3: the coupled pair on a grid larger than L2
ncu --set full --clock-control none --import-source on -k regex:"k_collide_band|k_markers_fix|k_markers_skin" \
    -s 8 -c 2 -o $out/${tag}_c3_full $C3 > $out/${tag}_c3_ncu_full.log 2>&1
# c4: the pure-fluid K4 at 512^3
$C4 > $out/${tag}_c4_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_collide_fix" \
    -s 3 -c 1 -o $out/${tag}_c4_full $C4 > $out/${tag}_c4_ncu_full.log 2>&1
# c5: the batched env kernels (8 envs)
$C5 > $out/${tag}_c5_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"batch" \
    -s 6 -c 2 -o $out/${tag}_c5_full $C5 > $out/${tag}_c5_ncu_full.log 2>&1
ls -la $out/${tag}_*
