"""Loader for the in-tree CUDA library (``_lib/librsim.so``).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the product API fails with ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os

from . import abi

LIB_PATH = os.environ.get("RSIM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "librsim.so")

# every symbol include/rsim.h declares
EXPORTS = ("rs_abi_version", "rs_last_error", "rs_snapshot_size", "rs_scene_create", "rs_scene_destroy",
           "rs_batch_create", "rs_batch_destroy", "rs_batch_buffers", "rs_set_state", "rs_get_state", "rs_step",
           "rs_render", "rs_grasp", "rs_step_host", "rs_set_trace", "rs_scene_set_mesh", "rs_render_mesh", "rs_arm_action", "rs_env_step", "rs_env_step_host",
           "rs_nav_shape", "rs_nav_fields", "rs_nav_geodesic", "rs_nav_path", "rs_settle",
           "rs_sphere_cast", "rs_proprio", "rs_step_stats", "rs_set_env_order")


class NativeLibraryError(RuntimeError):
    pass


class RsimError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the host
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    vp, i32, i64, dbl, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint32
    L.rs_abi_version.restype = C.c_int
    L.rs_last_error.restype = C.c_char_p
    L.rs_snapshot_size.restype = i64
    L.rs_snapshot_size.argtypes = [i32, i32]
    L.rs_scene_create.argtypes = [C.POINTER(abi.rs_scene_desc), C.POINTER(vp)]
    L.rs_scene_destroy.argtypes = [vp]
    L.rs_batch_create.argtypes = [C.POINTER(vp), i32, vp, i32, C.POINTER(abi.rs_physics_config),
                                  C.POINTER(abi.rs_render_config), i32, C.POINTER(vp)]
    L.rs_batch_destroy.argtypes = [vp]
    L.rs_batch_buffers.argtypes = [vp, C.POINTER(abi.rs_buffers)]
    L.rs_set_state.argtypes = [vp, vp, i64, vp, i32, vp]
    L.rs_get_state.argtypes = [vp, vp, i64, vp, i32, vp]
    L.rs_step.argtypes = [vp, vp, vp, vp, dbl, i32, vp]
    L.rs_render.argtypes = [vp, u32, vp, vp, vp, vp]
    L.rs_grasp.argtypes = [vp, vp, vp]
    L.rs_step_stats.argtypes = [vp, vp, vp]
    L.rs_set_env_order.argtypes = [vp, i32]
    L.rs_step_host.argtypes = [vp, vp, vp, dbl, i32, u32, vp, vp, vp, vp, vp]
    L.rs_set_trace.argtypes = [vp, vp, vp, i32, i32]
    L.rs_scene_set_mesh.argtypes = [vp, C.POINTER(abi.rs_mesh_desc)]
    L.rs_render_mesh.argtypes = [vp, u32, vp, vp, vp, vp]
    L.rsim_bench_render_exact.argtypes = [vp, u32, vp, vp, vp, vp]
    L.rsim_bench_env_cycles.argtypes = [vp, vp]
    L.rsim_bench_force_heavy.argtypes = [vp, C.c_int]
    L.rsim_bench_phase_cycles.argtypes = [vp, vp]
    L.rsim_bench_render_work_detail.argtypes = [vp, u32, vp, vp]
    L.rs_arm_action.argtypes = [vp, vp, vp, vp, vp]
    L.rs_env_step.argtypes = [vp, vp, dbl, i32, vp]
    L.rs_env_step_host.argtypes = [vp, vp, dbl, i32, u32, vp, vp, vp, vp, vp]
    L.rs_settle.argtypes = [vp, vp, vp, i32, dbl, vp, vp, vp, vp, vp]
    L.rs_sphere_cast.argtypes = [vp, vp, vp, vp, vp, i32, vp, vp, vp]
    L.rs_proprio.argtypes = [vp, vp, vp, i32, vp, vp, vp]
    L.rs_nav_shape.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
    L.rs_nav_fields.argtypes = [vp, vp, vp, i32, vp, vp, vp]
    L.rs_nav_geodesic.argtypes = [vp, vp, vp, vp, vp, i32, vp, vp]
    L.rs_nav_path.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("rs_abi_version", "rs_last_error", "rs_snapshot_size", "rs_scene_destroy",
                        "rs_batch_destroy"):
            getattr(L, name).restype = C.c_int
    if L.rs_abi_version() != 1:
        raise NativeLibraryError("ABI version mismatch")
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().rs_last_error().decode(errors="replace")
        raise RsimError(f"{what} failed (code {rc}): {msg}")
