timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
for w in c3 c2 c1; do python bench.py --workload $w --steps 300 --warmup 10 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"; done
