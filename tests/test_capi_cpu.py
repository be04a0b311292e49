"""CPU-side checks of the boundary: liblgs.so loads and exports every symbol include/lgs.h
declares, the ctypes signatures match the header, and no-GPU calls fail cleanly."""
import ctypes as C
import os
import re

import pytest

from paper_2511_16144_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "lgs.h")).read()
    return sorted(set(re.findall(r"LGS_API\s+[\w\s\*]+?\b(lgs_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for s in ("lgs_render_forward", "lgs_render_backward", "lgs_ctx_create", "lgs_map_create",
              "lgs_debug_tile_keys", "lgs_debug_projected"):
        assert s in syms


def test_library_exports_every_header_symbol():
    L = _lib.load()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == header_symbols()


def test_struct_layouts():
    # the C structs are plain fixed-width layouts; sizes pinned so a header edit cannot drift silently
    assert C.sizeof(_lib.LgsRenderConfig) == 6 * 8
    assert C.sizeof(_lib.LgsCamera) == 4 * 8 + 3 * 8 + 4 * 8 + 2 * 4
    assert C.sizeof(_lib.LgsGaussians) == 8 + 4 + 4 + 6 * 8 + 8
    assert C.sizeof(_lib.LgsMapGrads) == 6 * 8 + 4 + 4


def test_defaults_match_reference():
    """renderer.hpp:15-22."""
    c = _lib.load().lgs_render_config_default()
    assert (c.near_plane, c.dilation, c.alpha_clamp, c.alpha_skip, c.transmittance_min, c.radius_sigma) == (
        0.01, 0.3, 0.99, 1.0 / 255.0, 1e-4, 3.0)


def test_flat_grad_size():
    assert _lib.load().lgs_grads_flat_size(500_000, 16, 3) == 500_000 * (3 + 4 + 3 + 1 + 48 + 16)


def test_ctx_create_without_gpu_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = _lib.load().lgs_ctx_create(0, None, C.byref(h))
    assert st == _lib.LGS_ENODEV
    assert _lib.load().lgs_last_error()


def test_version():
    assert b"sm_100a" in _lib.load().lgs_version()


def test_comm_unique_id_and_argument_checks():
    """lgs_comm_* (multi-view all-reduce): NCCL ids come from the dynamically loaded libnccl.so.2
    (no GPU needed); the GPU-side entry points reject missing contexts before touching CUDA."""
    L = _lib.load()
    a, b = _lib.LgsCommId(), _lib.LgsCommId()
    assert L.lgs_comm_unique_id(C.byref(a)) == _lib.LGS_OK
    assert L.lgs_comm_unique_id(C.byref(b)) == _lib.LGS_OK
    assert any(a.bytes) and bytes(a.bytes) != bytes(b.bytes)
    assert L.lgs_comm_unique_id(None) == _lib.LGS_EINVAL
    assert L.lgs_comm_init(None, 2, 0, C.byref(a)) == _lib.LGS_EINVAL
    assert L.lgs_allreduce_f32(None, None, 0) == _lib.LGS_EINVAL
    assert L.lgs_allreduce_grads(None, None, None) == _lib.LGS_EINVAL
    assert L.lgs_comm_destroy(None) == _lib.LGS_EINVAL
