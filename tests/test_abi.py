"""The C-ABI library loads without a GPU and exports every symbol that
include/lpic_b200.h declares; GPU entry points fail loudly without CUDA."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lpic_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lpic_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_symbols():
    from paper_2212_01185_b200 import _native
    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_all_symbols():
    from paper_2212_01185_b200 import _native
    L = _native.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.lpic_version() == 1


def test_library_is_sm100a():
    """The shipped .so carries sm_100a SASS (cuobjdump), not just PTX."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    from paper_2212_01185_b200 import _native
    out = subprocess.run([exe, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_fnv_without_gpu():
    from paper_2212_01185_b200 import _native
    L = _native.load()
    buf = C.create_string_buffer(b"foobar", 6)
    assert L.lpic_fnv1a64(buf, 6) == 0x85944171f73967e8


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2212_01185_b200 as P
    from paper_2212_01185_b200._native import NativeUnavailable
    from conftest import make_weights
    w, cfg = make_weights("small", "glorot", 7)
    with pytest.raises(NativeUnavailable):
        P.encode(np.zeros((4, 4, 3), np.uint8), w, cfg, "wave")
    with pytest.raises(NativeUnavailable):
        P.forward_full(np.zeros((4, 4, 3), np.float32), w, cfg)


def test_status_and_precision_constants_match_header():
    """The Python layer's status / precision codes equal the header's #defines."""
    from paper_2212_01185_b200 import _native
    src = open(os.path.join(ROOT, "include", "lpic_b200.h")).read()
    defs = dict(re.findall(r"#define\s+(LPIC_[SP][A-Z_]*)\s+(\d+)", src))
    for name in ("LPIC_S_OK", "LPIC_S_NONFINITE", "LPIC_S_CORRUPT", "LPIC_S_CAPACITY", "LPIC_S_INTERNAL"):
        assert name in defs, name
        if hasattr(_native, name):
            assert getattr(_native, name) == int(defs[name]), name
    assert int(defs["LPIC_PREC_COMPAT"]) == 0 and int(defs["LPIC_PREC_FAST"]) == 1


@pytest.mark.parametrize("K,Cf,L,h,why", [
    (17, 16, 4, 2, "mixtures"),       # the reference accepts any K >= 1 that fits a byte (network.py:49-59)
    (3, 129, 4, 2, "filters"),
    (3, 16, 4, 4, "kernel_half"),
    (3, 16, 2, 2, "layers"),
    (0, 16, 4, 2, "mixtures"),
])
def test_config_range_refused_loudly(K, Cf, L, h, why):
    """The GPU build covers K <= 16, C <= 128, h <= 3, L >= 3 (every config
    of the reference's tests and BASELINE); outside that range model
    creation fails with a message before any device work -- never a silent
    fallback.  Checked through the C-ABI without a GPU."""
    from paper_2212_01185_b200 import _native
    Lb = _native.load()
    T = (2 * h + 1) * h + h
    arrs = [np.zeros(n, np.float32) for n in (T * 3 * Cf, Cf, max(L - 2, 1) * Cf * Cf, max(L - 2, 1) * Cf,
                                              12 * max(K, 1) * Cf, 12 * max(K, 1))]
    out = C.c_void_p()
    rc = Lb.lpic_model_create(*[a.ctypes.data for a in arrs], K, Cf, L, h, 0, C.byref(out))
    assert rc in (_native.LPIC_E_UNSUPPORTED, _native.LPIC_E_ARG)
    assert why.split("_")[0] in Lb.lpic_last_error().decode() or "layers" in Lb.lpic_last_error().decode()
    assert not out.value
