mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
python bench.py --impl reference --steps 2 --warmup 1 --cpu-sample 64 > gpurun_out/bench_ref1.json 2>&1; echo ref_rc=$?
cat gpurun_out/bench_ref1.json | tail -2
nproc
