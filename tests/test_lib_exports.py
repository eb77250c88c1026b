"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/uwsplat_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2411_19588_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uwsplat_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|uint64_t|const char\*)\s+(uws_\w+)\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libuwsplat_b200.so is not built (run `make` / __graft_entry__.build())")
    return _lib.load()


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_all_symbols_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.uws_version()
    assert isinstance(lib.uws_last_error(), bytes)


def test_workspace_queries_and_argument_errors(lib):
    n = ctypes.c_size_t(0)
    assert lib.uws_preprocess_workspace_size(1000, ctypes.byref(n)) == 0 and n.value > 0
    a, b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.uws_bin_workspace_size(1000, 5000, 8, 8, ctypes.byref(a), ctypes.byref(b)) == 0
    assert a.value > 0 and b.value > 0
    assert lib.uws_loss_workspace_size(32, 32, 3, ctypes.byref(n)) == 0
    # invalid arguments are rejected before touching the device
    assert lib.uws_preprocess_workspace_size(-1, ctypes.byref(n)) == _lib.UWS_EINVAL
    assert b"bad argument" in lib.uws_last_error()
    assert lib.uws_loss_fwd_bwd(None, None, 4, 4, 3, None, 0, 0.3, 0.1, None, None, None, None,
                                0, None) == _lib.UWS_EINVAL
    with pytest.raises(ValueError):
        _lib.call("uws_preprocess_workspace_size", -5, ctypes.byref(n))


def test_struct_layouts_match_header():
    # offsets the kernels rely on (uws_splat is 48 bytes, camera doubles 8-aligned)
    assert ctypes.sizeof(_lib.CameraC) == 8 + 4 * 8 + 9 * 8 + 3 * 8 + 2 * 8
    assert ctypes.sizeof(_lib.CloudC) == 6 * 8
    assert ctypes.sizeof(_lib.ProjectedC) == 9 * 8
    # 11 pointers, int32 cap + padding, 2 fix-up pointers
    assert ctypes.sizeof(_lib.RasterOutC) == 11 * 8 + 8 + 3 * 8   # + fix_pixels, fix_count, tile_order
    assert ctypes.sizeof(_lib.AdamParamsC) == 45 * 8


def test_pdl_launched_kernels_wait_first():
    """Every kernel launched with programmatic dependent launch (launch(...)) starts
    with pdl_entry() -- a PDL-launched kernel that does not wait could read its
    predecessor's outputs early -- and kernels launched serially need not."""
    import glob
    import re
    src = ""
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2411_19588_b200", "csrc", "*.cu*"))):
        src += open(f).read() + "\n"
    launched = {k for k in re.findall(r"[^_\w]launch\((?:\w+::)*(\w+)", src) if k.startswith("k_")}
    assert len(launched) >= 15
    bodies = {}
    for m in re.finditer(r"__global__\s+void\s+(?:__launch_bounds__\([^)]*\)\s*)?(\w+)\s*\([^;{]*?\)\s*\{",
                         src, flags=re.S):
        bodies.setdefault(m.group(1), []).append(src[m.end():m.end() + 200])
    for name in launched:
        assert name in bodies, name
        for b in bodies[name]:
            first = b.strip().split(";")[0]
            assert first == "pdl_entry()", (name, first)
