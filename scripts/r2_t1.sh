#!/bin/bash
# wide-row kernel on one-tile rows (F = 128) as tuning variants: parity + products / arxiv timings
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_affine.py tests/test_gpu_device.py tests/test_gpu_layer.py -m gpu -q -x -k "affine or feature or wide or q8 or layer" 2>&1 | tail -2
for cfg in products arxiv pubmed; do
  for v in 0 46 48 49; do
    timeout 300 python bench.py --config $cfg --dtype int8 --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg int8 v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done
  for dt in int8-row int8-feature; do for v in 0 56 57; do
    timeout 300 python bench.py --config $cfg --dtype $dt --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg $dt v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done; done
done
