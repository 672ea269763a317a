#!/bin/bash
# compute-sanitizer over scripts/sanitize_probe.py (every kernel family, small shapes).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize probe done' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
