#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_affine.py tests/test_gpu_device.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
for cfg in products reddit pubmed arxiv; do for v in 0 54; do
  timeout 300 python bench.py --config $cfg --dtype int8-row --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg row v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
done; done
