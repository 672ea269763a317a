#!/bin/bash
# Round-2 verification pass: GPU tests, smoke, bench lines (f32 / int8 / affine int8 / reference).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -16 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
for dt in int8 int8-row int8-feature; do
  timeout 300 python bench.py --dtype $dt --no-cpu-baseline > gpurun_out/bench_$dt.json 2> gpurun_out/bench_$dt.err; cat gpurun_out/bench_$dt.json; tail -2 gpurun_out/bench_$dt.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
