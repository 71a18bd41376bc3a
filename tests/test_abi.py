"""C-ABI library: loads on a CPU-only host and exports every symbol
include/rsim.h declares (no compute calls without a GPU)."""
import ctypes as C
import os
import re

from paper_2106_14405_b200 import abi, native
from paper_2106_14405_b200.state import snapshot_size

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = native.lib()
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(native.EXPORTS)


def test_abi_version_and_snapshot_size():
    L = native.lib()
    assert L.rs_abi_version() == 1
    assert L.rs_snapshot_size(42, 11) == snapshot_size(42, 11) == 7770  # 7,770 B


def test_struct_layouts_match_header():
    # field counts / sizes of the ctypes mirror (guards against header drift)
    assert C.sizeof(abi.rs_render_config) == 4 + 4 + 8 * 4
    assert C.sizeof(abi.rs_physics_config) == 144  # 15 doubles + 4 int32 with natural alignment
    names = [f[0] for f in abi.rs_scene_desc._fields_]
    hdr = open(os.path.join(ROOT, "include", "rsim.h")).read()
    body = hdr[hdr.index("typedef struct {"):hdr.index("} rs_scene_desc;")]
    for n in names:
        assert re.search(r"\b" + n + r"\b", body), n


def test_no_cpu_fallback():
    """The product refuses to run without CUDA instead of silently falling back."""
    import pytest
    import torch

    from paper_2106_14405_b200.sim import BatchSimulator

    with pytest.raises(native.NativeLibraryError):
        BatchSimulator(device="cpu")
    if not torch.cuda.is_available():
        with pytest.raises(Exception):
            BatchSimulator(device="cuda")
