#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python scripts/layer_probe.py 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --dtype int8 --no-cpu-baseline > gpurun_out/bench_int8.json 2> gpurun_out/bench_int8.err; cat gpurun_out/bench_int8.json
