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
timeout 300 python tools/idle_phases.py > $O/${T}_idle_phases.txt 2>&1; echo "idle_phases rc=$?"; tail -1 $O/${T}_idle_phases.txt
timeout 300 python tools/physics_only.py > $O/${T}_config2.jsonl 2>/dev/null; echo "physics_only rc=$?"
timeout 300 python tools/render_work.py > $O/${T}_render_work.txt 2>&1; echo "render_work rc=$?"
# summaries on the box (gpurun copies back <= 64 MiB): keep only the idle report
for m in idle interact mesh; do
  python tools/ncu_summary.py --lines $O/${T}_$m.ncu-rep > $O/${T}_full_$m.txt 2>&1
  python tools/ncu_summary.py --json $O/${T}_$m.ncu-rep > $O/${T}_kernels_$m.json 2>&1
done
python tools/ncu_summary.py --launches $O/${T}_launches.csv > $O/${T}_launches.txt 2>&1
rm -f $O/${T}_interact.ncu-rep $O/${T}_mesh.ncu-rep
du -sh $O
