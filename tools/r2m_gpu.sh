# mesh-path A/B: configs[3] sweep, default vs _lib_base (mesh + proxy ms per batch)
for r in 1 2; do
for V in default paper_2106_14405_b200/_lib_base; do
  if [ "$V" = default ]; then LIBV=""; else LIBV="$V/librsim.so"; fi
  RSIM_LIB=$LIBV KS=${KS:-3,7,12} timeout 600 python tools/render_sweep.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$V', d['k'], d['triangles_per_scene'], 'mesh ms', round(d['ms_per_batch_mesh'],3), 'proxy ms', round(d['ms_per_batch_proxy'],3))"
done
done
