#!/bin/bash
# compute-sanitizer over both probes (round-1 kernel families + round-2 additions)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for probe in sanitize_probe sanitize_probe_r2; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 \
        python scripts/$probe.py > gpurun_out/${probe}_$tool.log 2>&1
    echo "$probe $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|probe.*done' gpurun_out/${probe}_$tool.log | tr '\n' ' ')"
  done
done
