for v in 0 2 1.5 1 0.5; do
  export FSG_KM_PER_SM=$v
  echo "== KM_PER_SM $v" >> gpurun_out/sweep.txt
  python scripts/probe_timeline.py c2 --flush 2>&1 | tail -3 >> gpurun_out/sweep.txt
  for w in c2 c1 c3; do
    python bench.py --workload $w --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/sweep.txt
  done
done
FSG_KM_PER_SM=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_km1.log 2>&1
