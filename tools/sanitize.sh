#!/bin/bash
# compute-sanitizer over tools/san_case.py (every stage-kernel family, multi-tile pipelines):
# memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse), initcheck.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/san_case.py > gpurun_out/san_$tool.log 2>&1
  echo "exit $?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|Uninitialized|error" gpurun_out/san_$tool.log | sort | uniq -c | head -20
done
