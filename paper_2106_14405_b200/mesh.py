"""Triangle-soup scene path (BASELINE configs[3]).

``AssetDef.visual_mesh`` (scene.py:63-76) turns every collision proxy into a
triangle soup: boxes and hulls through their qhull triangulation, spheres as
10-gon prisms (radius r, height 2r).  For the 10k-200k-triangle render sweep
every planar triangle is subdivided into k x k sub-triangles:
the surface is unchanged, so the proxy ray caster over the same convex
shapes (spheres replaced by their prisms) stays the exact oracle.

Per part the soup is kept in the part's local frame (instanced: one copy per
layout, shared by all envs) with a bounding-volume hierarchy built here on
the host: median split on the longest centroid axis, <= 4 triangles per leaf,
depth-first flattened (an internal node's left child follows it, the right
child index is stored).  Node boxes are float32 rounded outward.
"""

from __future__ import annotations

import os

import numpy as np

from . import assets as A

LEAF = int(os.environ.get("RSIM_BVH_LEAF", "4"))  # triangles per leaf (env override: experiments)


def part_triangles(prim) -> np.ndarray:
    """[T, 3, 3] float64 triangles of one primitive in its part frame."""
    if prim.kind == A.KIND_SPHERE:
        hull = A.prism(prim.radius, 2 * prim.radius, 10)
    elif prim.kind == A.KIND_BOX:
        hull = A.Hull(prim.vertices)
    else:
        hull = prim
    return hull.vertices[hull.triangles]


def subdivide(tris: np.ndarray, k: int) -> np.ndarray:
    """Split every triangle into k*k coplanar sub-triangles (barycentric grid)."""
    if k <= 1:
        return tris
    out = []
    for a, b, c in tris:
        e1, e2 = (b - a) / k, (c - a) / k

        def P(i, j):
            return a + e1 * i + e2 * j

        for i in range(k):
            for j in range(k - i):
                out.append([P(i, j), P(i + 1, j), P(i, j + 1)])
                if i + j < k - 1:
                    out.append([P(i + 1, j), P(i + 1, j + 1), P(i, j + 1)])
    return np.asarray(out)


def build_bvh(tris: np.ndarray, first_tri: int):
    """Flattened BVH over `tris` (indices offset by first_tri).

    Returns (lo [N,3] f32, hi [N,3] f32, meta [N,2] i32, order): meta =
    (tri_first, tri_count) for leaves, (right_child, -1) for internal nodes;
    `order` permutes the triangles into leaf order."""
    cent = tris.mean(axis=1)
    tlo, thi = tris.min(axis=1), tris.max(axis=1)
    lo, hi, meta, order = [], [], [], []

    def rec(idx):
        node = len(meta)
        blo, bhi = tlo[idx].min(axis=0), thi[idx].max(axis=0)
        lo.append(np.nextafter(blo.astype(np.float32), np.float32(-np.inf)))
        hi.append(np.nextafter(bhi.astype(np.float32), np.float32(np.inf)))
        meta.append([0, 0])
        if len(idx) <= LEAF:
            meta[node] = [first_tri + len(order), len(idx)]
            order.extend(idx.tolist())
            return node
        c = cent[idx]
        ax = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
        srt = idx[np.argsort(c[:, ax], kind="stable")]
        h = len(srt) // 2
        rec(srt[:h])
        right = rec(srt[h:])
        meta[node] = [right, -1]
        return node

    rec(np.arange(len(tris)))
    return np.array(lo, np.float32), np.array(hi, np.float32), np.array(meta, np.int32), np.array(order, np.int64)


def compile_mesh(world, k: int = 1) -> dict:
    """Mesh tables for every part of `world` (same part order as compile_world)."""
    tri_all, lo_all, hi_all, meta_all = [], [], [], []
    part_node, part_bound = [0], []
    n_tri = 0
    for b in world.bodies:
        for _local, prim in b.parts:
            tris = subdivide(part_triangles(prim), k)
            lo, hi, meta, order = build_bvh(tris, n_tri)
            base = part_node[-1]
            meta = meta.copy()
            internal = meta[:, 1] < 0
            meta[internal, 0] += base
            tri_all.append(tris[order])
            lo_all.append(lo)
            hi_all.append(hi)
            meta_all.append(meta)
            part_node.append(base + len(meta))
            part_bound.append(float(np.sqrt((tris.reshape(-1, 3) ** 2).sum(axis=1)).max()))
            n_tri += len(tris)
    tri = np.concatenate(tri_all)
    tri = np.concatenate([tri[:, 0], tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]], axis=1)  # v0, e1, e2
    return {
        "tri": np.ascontiguousarray(tri, dtype=np.float64),
        "node_lo": np.concatenate(lo_all), "node_hi": np.concatenate(hi_all),
        "node_meta": np.concatenate(meta_all).astype(np.int32),
        "part_node_begin": np.array(part_node, np.int32),
        "part_bound": np.array(part_bound, np.float64),
        "k": int(k), "n_tri": int(n_tri),
    }


def prism_world(world):
    """Copy of `world` whose sphere parts are replaced by their 10-gon prisms
    (the convex oracle of the triangle path)."""
    import copy

    w = copy.copy(world)
    w.bodies = []
    for b in world.bodies:
        nb = copy.copy(b)
        nb.parts = [(local, A.prism(p.radius, 2 * p.radius, 10) if p.kind == A.KIND_SPHERE else p)
                    for local, p in b.parts]
        w.bodies.append(nb)
    return w


def k_for_triangles(world, target: int) -> int:
    base = sum(len(part_triangles(p)) for b in world.bodies for _, p in b.parts)
    return max(1, int(round(np.sqrt(target / base))))
