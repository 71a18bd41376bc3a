#!/bin/bash
# round-2 GPU pass: tests, bench, ncu full captures at HEAD, configs[3] sweep, sanitizers
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/r2b_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2b_gputest.log
timeout 400 python bench.py > $O/r2b_bench.json 2> $O/r2b_bench.err; echo "bench rc=$?"
tail -5 $O/r2b_bench.err
for m in idle interact mesh; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -f -o $O/r2b_$m python tools/ncu_targets.py $m > $O/r2b_ncu_$m.log 2>&1; echo "ncu $m rc=$?"
done
KS=3,7,12 timeout 600 python tools/render_sweep.py > $O/r2b_sweep.jsonl 2> $O/r2b_sweep.err; echo "sweep rc=$?"
for t in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_targets.py > $O/r2b_san_$t.log 2>&1; echo "sanitizer $t rc=$?"
  tail -3 $O/r2b_san_$t.log
done
