for mk in skinned host; do
python bench.py --workload c5 --markers $mk --no-cpu-baseline 2>gpurun_out/c5_$mk.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $mk', d['value'], d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value'], d['status'])" >> gpurun_out/c5.txt
done
