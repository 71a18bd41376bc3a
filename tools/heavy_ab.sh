python tools/traj_profile.py --interact --steps 20 > /dev/null 2>&1
for L in default paper_2106_14405_b200/_lib_pa; do
  if [ "$L" = default ]; then X=""; else X="$L/librsim.so"; fi
  for r in 0 1 5; do RSIM_LIB=$X python tools/heavy_replay.py --n 1 --rank $r --reps 3 --phase-rep 1 2>&1 | grep "rep 2" | sed "s|^|$L r$r |"; done
done
