cd $GRAFT_REPO_ROOT
nproc; lscpu | grep "Model name"
python -m pytest tests -m gpu -q 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --steps 20 --warmup 5 --dtype int8 --no-e2e --no-cpu-baseline > gpurun_out/bench_int8.json 2>&1; cat gpurun_out/bench_int8.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_wide -s 2 -c 1 -o gpurun_out/prof_spmm python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
