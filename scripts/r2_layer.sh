#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_device.py tests/test_gpu_parity.py tests/test_gpu_affine.py -m gpu -q -x 2>&1 | tail -5
timeout 300 python scripts/layer_probe.py 2>&1 | tail -5
bash scripts/ncu_capture.sh layer "gcn_layer_fused" 2 1 -- python scripts/layer_probe.py products
python scripts/ncu_raw_summary.py gpurun_out/ncu_layer_raw.csv --json > gpurun_out/ncu_layer_summary.json
