#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/gemm_probe.py 2>&1 | tail -3
timeout 300 python scripts/layer_probe.py 2>&1 | tail -3
bash scripts/ncu_capture.sh gemm2 "gemm_ordered_kernel" 2 1 -- python scripts/gemm_probe.py
python scripts/ncu_raw_summary.py gpurun_out/ncu_gemm2_raw.csv --json > gpurun_out/ncu_gemm2_summary.json
bash scripts/ncu_capture.sh layer2 "gcn_layer_fused" 2 1 -- python scripts/layer_probe.py products
python scripts/ncu_raw_summary.py gpurun_out/ncu_layer2_raw.csv --json > gpurun_out/ncu_layer2_summary.json
