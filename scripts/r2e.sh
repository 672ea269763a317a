cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python scripts/plan_probe.py products 2>&1 | tail -4
for cfg in products reddit pubmed; do for dt in f32 int8 int8-row int8-feature; do
  timeout 300 python bench.py --config $cfg --dtype $dt --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > gpurun_out/b_${cfg}_$dt.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b_${cfg}_$dt.json'));print('$cfg $dt', d['ms_per_step'], d['roofline']['frac'])"
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:row_scan_kernel|sample_fill_kernel|row_tile_total" -s 9 -c 3 -o gpurun_out/prof_sampler3 -f python scripts/plan_probe.py products > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:spmm_q8a" -s 2 -c 1 -o gpurun_out/prof_q8a2 -f python bench.py --dtype int8-row --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:spmm_q8_batch" -s 2 -c 1 -o gpurun_out/prof_q8b -f python bench.py --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:spmm_q8_batch" -s 2 -c 1 -o gpurun_out/prof_q8b_reddit -f python bench.py --config reddit --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
ls gpurun_out
