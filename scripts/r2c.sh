cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python scripts/plan_probe.py products 2>&1 | tail -4
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:row_scan_kernel|sample_fill_kernel" -s 6 -c 2 -o gpurun_out/prof_sampler -f python scripts/plan_probe.py products > gpurun_out/ncu_sampler.log 2>&1; tail -2 gpurun_out/ncu_sampler.log
