mkdir -p gpurun_out
python -m pytest tests/test_gpu_permute.py -q -x 2>&1 | tail -1
python bench.py --workload permute --steps 3 --warmup 3 > gpurun_out/r1e_permute.json 2>gpurun_out/perm5.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r1e_permute.json')); print(d['value'], d['roofline']['frac']); print(json.dumps(d['per_size']))"
python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_1811_09599_b200 import tensor_core as tc
n=16**7; src=torch.randn(n,dtype=torch.complex64,device='cuda'); dst=torch.empty_like(src)
for perm in [(0,1,3,4,6,2,5),(0,1,2,4,6,3,5),(0,2,3,4,6,1,5),(0,1,2,3,6,4,5)]:
    for _ in range(3): tc.permute_buffer(src,[16]*7,perm,out=dst)
    torch.cuda.synchronize(); a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): tc.permute_buffer(src,[16]*7,perm,out=dst)
    b.record(); torch.cuda.synchronize(); ms=a.elapsed_time(b)/5; print(perm, round(16*n/ms/1e6), 'GB/s')
"
