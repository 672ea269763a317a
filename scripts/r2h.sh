cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in products reddit pubmed arxiv; do for dt in int8 int8-feature; do
  timeout 300 python bench.py --config $cfg --dtype $dt --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err; python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg $dt', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/b.err
done
timeout 300 python bench.py --config $cfg --dtype int8 --variant 36 --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg int8 old-batch', d['ms_per_step'], d['roofline']['frac'])"
done
bash scripts/ncu_capture.sh q8t "spmm_q8t" 2 1 -- python bench.py --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
bash scripts/ncu_capture.sh q8t_reddit "spmm_q8t" 2 1 -- python bench.py --config reddit --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
du -sh gpurun_out
