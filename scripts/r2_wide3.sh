#!/bin/bash
# wide-row int8 kernel: exact + per-feature fast mode, parity + tuning + ncu
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device.py tests/test_gpu_affine.py -m gpu -q -x -k "wide or q8_schedules or every_spmm or affine or feature" 2>&1 | tail -3
for w in 32 64; do
  for v in 0 46 48 49 30; do
    timeout 300 python bench.py --config reddit --width $w --dtype int8 --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('reddit W$w int8 v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done
  for v in 0 55; do
    timeout 300 python bench.py --config reddit --width $w --dtype int8-feature --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('reddit W$w int8-feature v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done
bash scripts/ncu_capture.sh q8wide_feat "spmm_q8_wide" 2 1 -- python bench.py --config reddit --dtype int8-feature --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
python scripts/ncu_raw_summary.py gpurun_out/ncu_q8wide_feat_raw.csv --json > gpurun_out/ncu_q8wide_feat_summary.json
head -c 1200 gpurun_out/ncu_q8wide_feat_summary.json
