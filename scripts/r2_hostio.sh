#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hostio.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_ref_suite.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));e=d['e2e'];print(d['ms_per_step'], e['ms_per_step'], e['sync_call'], e['pybind_call'])"
