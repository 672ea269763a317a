#!/bin/bash
# closing pass after the rolled wide-row kernel: ncu captures of its three
# decodes on reddit, then the r2_final2.sh verification
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
B="python bench.py --config reddit --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer"
bash scripts/ncu_capture.sh q8wide "spmm_q8_wide" 2 1 -- $B --dtype int8
bash scripts/ncu_capture.sh q8wide_feat "spmm_q8_wide" 2 1 -- $B --dtype int8-feature
bash scripts/ncu_capture.sh q8wide_row "spmm_q8_wide" 2 1 -- $B --dtype int8-row
for n in q8wide q8wide_feat q8wide_row; do python scripts/ncu_raw_summary.py gpurun_out/ncu_${n}_raw.csv --json > gpurun_out/ncu_${n}_summary.json; done
bash scripts/r2_final2.sh
