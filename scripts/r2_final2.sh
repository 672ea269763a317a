#!/bin/bash
# Round-2 closing verification with the wide-row int8 kernel: every GPU test,
# smoke, bench lines (products f32 / int8 / affine, reddit int8 / affine,
# reference), configs table, timed-region launch list.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -14 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
for dt in int8 int8-row int8-feature; do
  timeout 300 python bench.py --dtype $dt --no-cpu-baseline --no-layer > gpurun_out/bench_$dt.json 2> gpurun_out/bench_$dt.err; tail -1 gpurun_out/bench_$dt.err
  timeout 300 python bench.py --config reddit --dtype $dt --no-layer > gpurun_out/bench_reddit_$dt.json 2> gpurun_out/bench_reddit_$dt.err; tail -1 gpurun_out/bench_reddit_$dt.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_timed.csv > gpurun_out/launches_timed_summary.json
for f in bench bench_int8 bench_int8-row bench_int8-feature bench_reddit_int8 bench_reddit_int8-row bench_reddit_int8-feature bench_ref; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d.get('ms_per_step'), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('ms_per_step'))"; done
timeout 1500 python scripts/measure_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
