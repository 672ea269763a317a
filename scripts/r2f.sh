cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_affine.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_device.py -m gpu -q -x 2>&1 | tail -3
for cfg in products reddit pubmed; do for dt in f32 int8 int8-row int8-feature; do
  timeout 300 python bench.py --config $cfg --dtype $dt --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg $dt', d['ms_per_step'], d['roofline']['frac'])"
done; done
bash scripts/ncu_capture.sh q8a "spmm_q8a" 2 1 -- python bench.py --dtype int8-row --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
bash scripts/ncu_capture.sh q8b "spmm_q8_batch" 2 1 -- python bench.py --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
bash scripts/ncu_capture.sh q8b_reddit "spmm_q8_batch" 2 1 -- python bench.py --config reddit --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
bash scripts/ncu_capture.sh sampler "row_scan_kernel|sample_fill_kernel|row_tile_total" 9 3 -- python scripts/plan_probe.py products
du -sh gpurun_out
