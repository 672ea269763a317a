#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python scripts/sanitize_probe_r2.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_probe_r2.py > gpurun_out/sanitize_r2_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|probe r2 done' gpurun_out/sanitize_r2_$tool.log | tr '\n' ' ')"
done
