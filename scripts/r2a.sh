cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nvidia-smi -L
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --dtype int8 --no-cpu-baseline > gpurun_out/bench_int8.json 2>&1; cat gpurun_out/bench_int8.json
