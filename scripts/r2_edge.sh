#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_gpu_device.py -m gpu -q -x -k "edge_shapes or wide" 2>&1 | tail -15
