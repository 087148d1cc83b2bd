for w in c2 c1 c3; do for mk in skinned host; do
python bench.py --workload $w --markers $mk --steps 300 --warmup 10 --e2e-steps 50 --no-cpu-baseline 2>gpurun_out/err_$w_$mk.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $mk', d['value'], d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value'], d['status'])" >> gpurun_out/skinbench.txt
done; done
