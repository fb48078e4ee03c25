#!/bin/bash
# compute-sanitizer passes over scripts/sanitize_cases.py; logs to gpurun_out/sanitize_*.log
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
