#!/bin/bash
# Round-2 measurement pass with every current default kernel: configs, shard
# scaling, PCIe ceilings, launch list of the timed region, ncu captures.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python scripts/measure_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
timeout 600 python scripts/shard_scaling.py products > gpurun_out/shard_scaling_products.json 2>/dev/null
timeout 600 python scripts/shard_scaling.py reddit > gpurun_out/shard_scaling_reddit.json 2>/dev/null
timeout 300 python scripts/measure_pcie.py > gpurun_out/pcie.json 2>/dev/null
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_timed.csv > gpurun_out/launches_timed_summary.json
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_timed_int8.csv python bench.py --dtype int8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_timed_int8.csv > gpurun_out/launches_timed_int8_summary.json
B="python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer"
bash scripts/ncu_capture.sh q8r_row "spmm_q8r" 2 1 -- $B --dtype int8-row
bash scripts/ncu_capture.sh q8r_feat "spmm_q8r" 2 1 -- $B --dtype int8-feature
bash scripts/ncu_capture.sh q8b_reddit "spmm_q8_batch" 2 1 -- $B --config reddit --dtype int8
bash scripts/ncu_capture.sh q8r_feat_reddit "spmm_q8r" 2 1 -- $B --config reddit --dtype int8-feature
for f in gpurun_out/ncu_q8r_row_raw.csv gpurun_out/ncu_q8r_feat_raw.csv gpurun_out/ncu_q8b_reddit_raw.csv gpurun_out/ncu_q8r_feat_reddit_raw.csv; do
  python scripts/ncu_raw_summary.py $f --json > ${f%_raw.csv}_summary.json; done
ls gpurun_out | head -50
