#!/bin/bash
# small-graph int8: batch kernel vs wide-row kernel on one-tile rows, repeated
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2 3; do
for cfg in pubmed arxiv; do
  for dv in "f32 0" "int8 0" "int8 46" "int8 49" "int8 38" "int8 39"; do set -- $dv
    timeout 300 python bench.py --config $cfg --dtype $1 --variant $2 --no-cpu-baseline --no-e2e --no-layer --steps 50 --warmup 10 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg $1 v$2', d['ms_per_step'], d['gpu_launches_per_step']['kernels'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done; done
