#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layer.py -m gpu -q -x 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
python scripts/exact_probe.py 2>&1 | tail -4
