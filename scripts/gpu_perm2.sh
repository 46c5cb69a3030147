mkdir -p gpurun_out
python -m pytest tests/test_gpu_permute.py -q -x 2>&1 | tail -2
python bench.py --workload permute --steps 3 --warmup 3 > gpurun_out/perm2.json 2>gpurun_out/perm2.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/perm2.json')); print(d['value'], d['roofline']['frac']); print(json.dumps(d['per_size']))"
python scripts/step_profile.py auto 1024 2>&1 | grep permute
