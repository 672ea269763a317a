#!/bin/bash
# int8 wide-row kernel: parity (small + reddit config scale), variant timings, ncu capture
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device.py -m gpu -q -x -k "wide or q8_schedules or every_spmm" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "reddit" 2>&1 | tail -3
for w in 32 64; do
  for v in 0 46 48 49 30; do
    timeout 300 python bench.py --config reddit --width $w --dtype int8 --variant $v --no-cpu-baseline --no-e2e --no-layer --steps 20 --warmup 5 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.load(open('/tmp/b.json'));print('reddit W$w int8 v$v', d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done
timeout 300 python bench.py --config reddit --dtype int8 --no-layer > gpurun_out/r02_bench_reddit_int8.json 2>gpurun_out/r02_bench_reddit_int8.err
cat gpurun_out/r02_bench_reddit_int8.json
bash scripts/ncu_capture.sh q8wide "spmm_q8_wide" 2 1 -- python bench.py --config reddit --dtype int8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-layer
python scripts/ncu_raw_summary.py gpurun_out/ncu_q8wide_raw.csv --json > gpurun_out/ncu_q8wide_summary.json
head -c 1500 gpurun_out/ncu_q8wide_summary.json
