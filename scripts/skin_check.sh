timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1
rm -f gpurun_out/skinbench.txt; bash scripts/bench_markers.sh
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"skin|markers_fix|collide_band" -c 40 --csv --log-file gpurun_out/skin_launch.csv python bench.py --workload c2 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
