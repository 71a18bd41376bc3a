#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r2c_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2c_gputest.log
for t in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_targets.py > $O/r2c_san_$t.log 2>&1; echo "sanitizer $t rc=$?"
  tail -3 $O/r2c_san_$t.log
done
