#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/exact_probe.py 2>&1 | tail -4
for cfg in pubmed arxiv products; do
  timeout 300 python bench.py --config $cfg --dtype int8 --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg int8', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/b.err
done
bash scripts/ncu_capture.sh hub "spmm_hub_kernel" 0 2 -- python scripts/exact_probe.py arxiv
python scripts/ncu_raw_summary.py gpurun_out/ncu_hub_raw.csv --json > gpurun_out/ncu_hub_summary.json
