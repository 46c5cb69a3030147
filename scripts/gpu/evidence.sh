#!/bin/bash
# Round evidence run on one B200 (gpurun): GPU tests, smoke, the default bench
# line, the reference arm, and the secondary workloads.  Outputs -> gpurun_out/$TAG_*.
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference_arm.json 2> gpurun_out/${TAG}_reference_arm.err
echo done
