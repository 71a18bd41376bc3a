#!/bin/bash
# A/B: bench.py with the default library and with a variant (RSIM_LIB), alternating
# usage: tools/ab_bench.sh <variant_dir> <tag> [rounds]
V=$1; T=$2; R=${3:-2}
for r in $(seq 1 $R); do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_A$r.json 2>/dev/null; echo "A$r rc=$?"
  RSIM_LIB=$V/librsim.so timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_B$r.json 2>/dev/null; echo "B$r rc=$?"
done
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/${T}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        k=d["kernels_ms_per_step"]
        print(f, round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"],4), "inter", round(d["interact"]["value"]), "grasp", round(d["interact_grasp"]["value"]), "1cam", round(d["one_camera"]["value"]), "phys_alone", round(k["alone"]["ik+step+grasp"],4), "rend_alone", round(k["alone"]["render_kernel"],4))
    except Exception as e: print(f, "ERR", e)
PY
