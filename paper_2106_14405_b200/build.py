"""Build the in-tree CUDA library ``_lib/librsim.so`` for sm_100a.

Plain nvcc (no torch extension machinery): the library exposes only the
C-ABI of ``include/rsim.h``.  The physics and render units use FMA
contraction (physics: measured round 2, every discrete output -- pair lists,
contact counts, sleep flags, counters -- stays bit-exact against the oracle
and the reference goldens, states within 1e-12, and Interact runs 10 %
faster); nav, settle (GJK) and query keep ``-fmad=false``, where the
results are bit-exact against the reference.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.environ.get("RSIM_CSRC") or os.path.join(HERE, "csrc")  # RSIM_CSRC: A/B source tree
# RSIM_LIB_DIR / RSIM_NVCC_FLAGS: build an A/B variant elsewhere (e.g. _lib_w2 with
# -DRSIM_WARPS_PER_BLOCK=2), loaded with RSIM_LIB=<dir>/librsim.so
OUT_DIR = os.environ.get("RSIM_LIB_DIR") or os.path.join(HERE, "_lib")
EXTRA = os.environ.get("RSIM_NVCC_FLAGS", "").split()
LIB = os.path.join(OUT_DIR, "librsim.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
UNITS = {
    "physics.cu": [],  # FMA contraction (was -fmad=false)
    "render.cu": [],
    "abi.cu": [],
    "peak.cu": [],
    "nav.cu": ["-fmad=false"],
    "settle.cu": ["-fmad=false"],
    "query.cu": ["-fmad=false"],
}
HEADERS = ["device.cuh", "se3.cuh", "navgrid.cuh", "bulk.cuh"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    srcs = [os.path.join(CSRC, f) for f in list(UNITS) + HEADERS]
    srcs.append(os.path.join(HERE, "..", "include", "rsim.h"))
    srcs.append(os.path.join(HERE, "..", "include", "rsim_bench.h"))
    srcs.append(__file__)
    return any(os.path.getmtime(s) > t for s in srcs)


def _obj_stale(unit: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [os.path.join(CSRC, unit), __file__] + [os.path.join(CSRC, h) for h in HEADERS]
    deps += [os.path.join(HERE, "..", "include", h) for h in ("rsim.h", "rsim_bench.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the units that changed (in parallel), then link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = _nvcc()
    objs, cmds = [], []
    for unit, extra in UNITS.items():
        obj = os.path.join(OUT_DIR, unit.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _obj_stale(unit, obj):
            continue
        cmd = [nvcc, *ARCH, *COMMON, *extra, *EXTRA, "-c", os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c, check=True), cmds)):
            pass
    tmp = LIB + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
