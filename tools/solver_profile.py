"""Replay slow envs (gpurun_out/heavy_envs.npz from tools/traj_profile.py) on
an instrumented oracle build (-DORC_PROFILE) and report where the block LCP
spends its work: block sizes, active-set iterations, eigensolves (raw, and
after the GPU's 2-slot per-block cache), Jacobi sweeps.

    python tools/solver_profile.py [gpurun_out/heavy_envs.npz]
"""
import collections
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.oracle as O  # noqa: E402
from paper_2106_14405_b200.compiler import compile_world  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

PROF_LIB = "/tmp/orcprof/liboracle.so"
os.makedirs(os.path.dirname(PROF_LIB), exist_ok=True)
subprocess.run(["gcc", "-O2", "-fPIC", "-std=gnu99", "-ffp-contract=off", "-DORC_PROFILE", "-shared", "-o", PROF_LIB,
                os.path.join(ROOT, "oracle", "rsim_oracle.c"), "-lm", "-I", os.path.join(ROOT, "include")], check=True)
O.LIB = PROF_LIB
L = O.lib()
L.orc_profile_take.restype = C.c_int
L.orc_profile_take.argtypes = [C.c_void_p, C.c_int]
REC = 8

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "heavy_envs.npz")
d = np.load(path)
orcs = {}
seen = set()
for i in np.argsort(-np.abs(d["cycles"])):
    key = (int(d["env"][i]), int(d["step"][i]))
    if abs(d["cycles"][i]) < 1.5e6 or key in seen:
        continue
    seen.add(key)
    v = int(d["layout"][i])
    if v not in orcs:
        orcs[v] = O.Oracle(compile_world(build_world(v, flat_clutter())))
    orc = orcs[v]
    snap = d["pre"][i].tobytes()
    st = WorldState.from_bytes(snap)
    a = d["action"][i]
    nsj = len(st.joints) - 7
    tgt, _ = orc.apply_arm_action(st.joints[nsj:], a[:3])
    L.orc_profile_take(None, 0)
    r = orc.step(snap, tgt, a[4:6])
    buf = np.zeros((1 << 20, REC), np.int32)
    n = L.orc_profile_take(buf.ctypes.data, 1 << 20)
    recs = buf[:n]
    sub, it, g, m, na, mask, sweeps, asi = recs.T
    # the GPU eigen cache: 2 slots per (substep, group), keyed by mask, alternating replacement
    cache = {}
    misses = 0
    miss_sweeps = 0
    miss_na = []
    for s_, g_, mask_, sw, na_ in zip(sub, g, mask, sweeps, na):
        slots = cache.setdefault((s_, g_), [None, None, 0])
        if mask_ in slots[:2]:
            continue
        misses += 1
        miss_sweeps += sw
        miss_na.append(na_)
        slots[slots[2]] = mask_
        slots[2] ^= 1
    def sim_cache(nslots):  # LRU over (substep, group) blocks, keyed by the active mask
        lru, miss = {}, 0
        for s_, g_, mask_ in zip(sub, g, mask):
            q = lru.setdefault((s_, g_), [])
            if mask_ in q:
                q.remove(mask_)
            else:
                miss += 1
                if len(q) >= nslots:
                    q.pop(0)
            q.append(mask_)
        return miss
    lru_misses = {k: sim_cache(k) for k in (2, 4, 8, 16)}
    blocks = collections.Counter()
    for s_, it_, g_, m_ in zip(sub, it, g, m):
        blocks[(s_, it_, g_)] = m_
    print(f"env {key[0]:5d} step {key[1]:2d} {abs(d['cycles'][i]) / 1.965e3:7.0f} us | block solves "
          f"{len(blocks):4d} (m: {dict(collections.Counter(blocks.values()))}) | pinv calls {n:5d} "
          f"(na mean {na.mean() if n else 0:.1f}) sweeps/call {sweeps.mean() if n else 0:.1f} | "
          f"GPU-cache misses {misses} (na mean {np.mean(miss_na) if miss_na else 0:.1f}, sweeps {miss_sweeps}) | "
          f"AS iters/solve {n / max(1, len(blocks)):.1f} | LRU misses by slots {lru_misses}", flush=True)
