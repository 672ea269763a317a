#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device.py tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -x 2>&1 | tail -3
python scripts/plan_probe.py products 2>&1 | tail -4
for cfg in products reddit pubmed arxiv; do
  for vs in "0 0" "38 3" "39 3" "43 3" "44 3" "45 3"; do set -- $vs
    timeout 300 python bench.py --config $cfg --dtype int8 --variant $1 --sched $2 --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg int8 v$1 s$2', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done
bash scripts/ncu_capture.sh q8b38s3 "spmm_q8_batch" 2 1 -- python bench.py --dtype int8 --variant 38 --sched 3 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
python scripts/ncu_raw_summary.py gpurun_out/ncu_q8b38s3_raw.csv --json > gpurun_out/ncu_q8b38s3_summary.json
bash scripts/ncu_capture.sh sampler2 "row_scan_coop_kernel|sample_fill_kernel" 6 2 -- python scripts/plan_probe.py products
python scripts/ncu_raw_summary.py gpurun_out/ncu_sampler2_raw.csv --json > gpurun_out/ncu_sampler2_summary.json
