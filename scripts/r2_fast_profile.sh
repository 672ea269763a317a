#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer"
bash scripts/ncu_capture.sh q8f_feat "spmm_q8_batch" 2 1 -- $B --dtype int8-feature
bash scripts/ncu_capture.sh q8f_feat_reddit "spmm_q8_batch" 2 1 -- $B --config reddit --dtype int8-feature
bash scripts/ncu_capture.sh q8f_row "spmm_q8r" 2 1 -- $B --dtype int8-row
bash scripts/ncu_capture.sh q8f_row_reddit "spmm_q8_batch" 2 1 -- $B --config reddit --dtype int8-row
bash scripts/ncu_capture.sh layer_bcast "gcn_layer_fused" 2 1 -- python scripts/p2p_layer_probe.py
for f in gpurun_out/ncu_q8f_*_raw.csv gpurun_out/ncu_layer_bcast_raw.csv; do python scripts/ncu_raw_summary.py $f --json > ${f%_raw.csv}_summary.json; done
for dt in int8-row int8-feature; do
  timeout 300 python bench.py --dtype $dt --no-cpu-baseline --no-layer > gpurun_out/bench_$dt.json 2> gpurun_out/bench_$dt.err; tail -1 gpurun_out/bench_$dt.err
  timeout 300 python bench.py --config reddit --dtype $dt --no-cpu-baseline --no-layer --no-e2e > gpurun_out/bench_reddit_$dt.json 2> /dev/null
done
timeout 300 python bench.py --config reddit --dtype int8 --no-cpu-baseline --no-layer --no-e2e > gpurun_out/bench_reddit_int8.json 2> /dev/null
timeout 300 python bench.py --config reddit --no-cpu-baseline --no-layer --no-e2e > gpurun_out/bench_reddit_f32.json 2> /dev/null
ls gpurun_out/
