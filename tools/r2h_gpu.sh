set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
bash tools/ab_multi.sh r2aj 2 default paper_2106_14405_b200/_lib_base
for V in default paper_2106_14405_b200/_lib_base; do
  if [ "$V" = default ]; then LIBV=""; else LIBV="$V/librsim.so"; fi
  RSIM_LIB=$LIBV timeout 300 python tools/physics_only.py 2>/dev/null | tail -3
done
