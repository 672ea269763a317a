#!/bin/bash
# One GPU verification pass: tests, smoke, bench lines, ncu launch list + full captures.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --dtype int8 --no-cpu-baseline > gpurun_out/bench_int8.json 2>&1; cat gpurun_out/bench_int8.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
# launch list of the timed region only (NVTX range "timed")
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_all.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
for dt in f32 int8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:spmm_ring|spmm_q8_batch" -s 2 -c 1 -o /tmp/prof_spmm_$dt -f \
      python bench.py --steps 2 --warmup 2 --dtype $dt --no-e2e --no-cpu-baseline --no-layer > gpurun_out/ncu_$dt.log 2>&1; tail -1 gpurun_out/ncu_$dt.log
done
python scripts/shard_scaling.py products > gpurun_out/shard_scaling_products.json
python scripts/shard_scaling.py reddit > gpurun_out/shard_scaling_reddit.json
python scripts/measure_pcie.py > gpurun_out/pcie.json
python scripts/ncu_summary.py /tmp/prof_spmm_f32.ncu-rep /tmp/prof_spmm_int8.ncu-rep > gpurun_out/ncu_full_summary.json
python scripts/launch_summary.py gpurun_out/launches_timed.csv > gpurun_out/launches_timed_summary.json
python scripts/launch_summary.py gpurun_out/launches_all.csv > gpurun_out/launches_all_summary.json
ls -la gpurun_out
