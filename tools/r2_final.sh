#!/bin/bash
# round-2 measurement pass at HEAD: gpu tests, bench, ncu --set full of the four
# kernels (idle / interact / mesh workloads), launch list, sanitizers
O=gpurun_out; T=${1:-r2z}
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${T}_gputest.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
for m in idle interact mesh; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -f -o $O/${T}_$m python tools/ncu_targets.py $m > $O/${T}_ncu_$m.log 2>&1; echo "ncu $m rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_bench.log 2>&1; echo "launches rc=$?"
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_targets.py > $O/${T}_san_$t.log 2>&1; echo "sanitizer $t rc=$?"; tail -1 $O/${T}_san_$t.log
done
