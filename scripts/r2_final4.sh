#!/bin/bash
# last confirmation after the per-feature smem params: full GPU suite, smoke,
# reddit per-feature bench line + ncu capture, headline bench
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/ncu_capture.sh q8wide_feat "spmm_q8_wide" 2 1 -- python bench.py --config reddit --dtype int8-feature --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
python scripts/ncu_raw_summary.py gpurun_out/ncu_q8wide_feat_raw.csv --json > gpurun_out/ncu_q8wide_feat_summary.json
timeout 300 python bench.py --config reddit --dtype int8-feature --no-layer > gpurun_out/bench_reddit_int8-feature.json 2> gpurun_out/bench_reddit_int8-feature.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for f in bench bench_reddit_int8-feature; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d.get('ms_per_step'), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('ms_per_step'))"; done
