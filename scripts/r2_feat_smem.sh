#!/bin/bash
# per-feature wide-row epilogue with shared-memory params: parity + reddit timings
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_gpu_affine.py tests/test_gpu_device.py -m gpu -q -x -k "affine or feature or wide or q8" 2>&1 | tail -2
for w in 32 64; do for v in 0 56; do
  timeout 300 python bench.py --config reddit --width $w --dtype int8-feature --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('reddit W$w int8-feature v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
done; done
