#!/bin/bash
# A/B/C...: bench.py per library variant, alternating rounds
# usage: tools/ab_multi.sh <tag> <rounds> <lib_dir>...   ("default" = paper_2106_14405_b200/_lib)
T=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  i=0
  for V in "$@"; do
    i=$((i+1))
    if [ "$V" = default ]; then LIBV=""; else LIBV="$V/librsim.so"; fi
    RSIM_LIB=$LIBV timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_v${i}_r$r.json 2>/dev/null; echo "v$i r$r rc=$?"
  done
done
python - "$@" <<PY
import json,glob,sys
names=sys.argv[1:]
for f in sorted(glob.glob("gpurun_out/${T}_v*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        k=d["kernels_ms_per_step"]
        v=int(f.split("_v")[1].split("_")[0])
        print(f.split("/")[-1], names[v-1].split("/")[-1], round(d["value"]), "e2e", round(d["e2e"]["value"]), "inter", round(d["interact"]["value"]), "grasp", round(d["interact_grasp"]["value"]), "1cam", round(d["one_camera"]["value"]), "phys_alone", round(k["alone"]["ik+step+grasp"],4), "rend_alone", round(k["alone"]["render_kernel"],4), "p50us", round(d["physics_latency"]["p50_us"],1))
    except Exception as e: print(f, "ERR", e)
PY
