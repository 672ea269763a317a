#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scripts/plan_probe.py products 2>&1 | tail -4
python scripts/exact_probe.py 2>&1 | tail -4
for cfg in products reddit pubmed arxiv; do
  for dt in int8 int8-row int8-feature; do for v in 0 52 53; do
    [ "$dt" = "int8" ] && [ "$v" != "0" ] && continue
    timeout 300 python bench.py --config $cfg --dtype $dt --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg $dt v$v', d['ms_per_step'], d['roofline']['frac'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done; done
done
bash scripts/ncu_capture.sh sampler3 "row_scan_coop_kernel|sample_fill_kernel" 6 2 -- python scripts/plan_probe.py products
python scripts/ncu_raw_summary.py gpurun_out/ncu_sampler3_raw.csv --json > gpurun_out/ncu_sampler3_summary.json
bash scripts/ncu_capture.sh q8x "spmm_q8_batch" 2 1 -- python bench.py --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
python scripts/ncu_raw_summary.py gpurun_out/ncu_q8x_raw.csv --json > gpurun_out/ncu_q8x_summary.json
