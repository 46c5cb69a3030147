mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c2.json; python -c "import json;d=json.load(open('gpurun_out/b_c2.json'));print('c2 eager', d['value'], d['e2e']['value'], d['roofline'])"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --graph > gpurun_out/b_c2g.json; python -c "import json;d=json.load(open('gpurun_out/b_c2g.json'));print('c2 graph', d['value'], d['e2e']['value'])"
python bench.py --workload config1 --steps 20 --warmup 3 --cpu-sample 64 > gpurun_out/b_c1.json; python -c "import json;d=json.load(open('gpurun_out/b_c1.json'));print('c1 eager', d['value'], d['e2e']['value'], d['cpu_baseline']['value'])"
python bench.py --workload config1 --steps 20 --warmup 3 --no-cpu-baseline --graph > gpurun_out/b_c1g.json; python -c "import json;d=json.load(open('gpurun_out/b_c1g.json'));print('c1 graph', d['value'], d['e2e']['value'], d['gpu_launches'])"
python bench.py --workload config5 --paths 3 > gpurun_out/b_c5.json; cut -c 1-600 gpurun_out/b_c5.json
