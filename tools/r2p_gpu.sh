# physics A/B: bench (2 alternating rounds), configs[2] physics-only and idle phase clocks, default vs _lib_base
T=${1:-r2p}
bash tools/ab_multi.sh $T 2 default paper_2106_14405_b200/_lib_base 2>&1 | tail -4
for V in default paper_2106_14405_b200/_lib_base; do
  if [ "$V" = default ]; then LIBV=""; else LIBV="$V/librsim.so"; fi
  echo "== $V"
  RSIM_LIB=$LIBV timeout 300 python tools/physics_only.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['scenario'], round(d['env_steps_per_s']), d['latency_us'])"
  RSIM_LIB=$LIBV timeout 300 python tools/idle_phases.py 2>/dev/null | tail -1
done
