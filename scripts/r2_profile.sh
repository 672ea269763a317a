#!/bin/bash
# Round-2 profiling pass: timed-region launch list, ncu --set full captures of
# every kernel family (summarised on the box), probes, sanitizer.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer"
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_timed.csv > gpurun_out/launches_timed_summary.json; cat gpurun_out/launches_timed_summary.json | head -20
bash scripts/ncu_capture.sh f32 "spmm_ring_bal" 2 1 -- $B
bash scripts/ncu_capture.sh q8b "spmm_q8_batch" 2 1 -- $B --dtype int8
bash scripts/ncu_capture.sh q8r_row "spmm_q8r" 2 1 -- $B --dtype int8-row
bash scripts/ncu_capture.sh q8r_feat "spmm_q8r" 2 1 -- $B --dtype int8-feature
bash scripts/ncu_capture.sh f32_reddit "spmm_ring" 2 1 -- $B --config reddit
bash scripts/ncu_capture.sh q8b_reddit "spmm_q8_batch" 2 1 -- $B --config reddit --dtype int8
bash scripts/ncu_capture.sh sampler "row_scan_kernel|sample_fill_kernel|row_tile_total" 9 3 -- python scripts/plan_probe.py products
bash scripts/ncu_capture.sh exact "spmm_hub_kernel|spmm_ring_bal" 0 4 -- python scripts/exact_probe.py
bash scripts/ncu_capture.sh gemm "gemm_ordered_kernel|tc_gemm_kernel" 2 4 -- python scripts/gemm_probe.py
bash scripts/ncu_capture.sh quant "fit_partial|quantize_fast|dequantize_u8_flat" 3 3 -- python scripts/quant_probe.py
for f in gpurun_out/ncu_*_raw.csv; do python scripts/ncu_raw_summary.py $f --json > ${f%_raw.csv}_summary.json; done
python scripts/plan_probe.py products 2>&1 | tail -4
python scripts/exact_probe.py 2>&1 | tail -8
python scripts/gemm_probe.py 2>&1 | tail -4
python scripts/quant_probe.py 2>&1 | tail -4
bash scripts/sanitize.sh
du -sh gpurun_out
