# render A/B: render parity tests, work counters, bench default vs _lib_base
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "render or edges or properties or mesh or smoke or env" 2>&1 | tail -3
python tools/render_work.py 2>&1 | tail -12
bash tools/ab_multi.sh ${1:-r2ak} 2 default paper_2106_14405_b200/_lib_base
