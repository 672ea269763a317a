#!/bin/bash
# wide-row int8 kernel tuning + the full GPU suite
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for w in 32 64; do
  for v in 0 46 48 49; do
    timeout 300 python bench.py --config reddit --width $w --dtype int8 --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('reddit W$w int8 v$v', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_wide.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu_wide.log
