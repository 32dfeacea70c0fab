"""Host-only checks of the C ABI (no GPU needed): the library loads, exports every
function include/km.h declares, and rejects invalid arguments before any launch."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "km.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(km_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_api():
    names = declared_functions()
    for f in ["km_create", "km_assign", "km_update", "km_run", "km_destroy"]:
        assert f in names


def test_library_exports_every_declared_symbol():
    import paper_2412_02244_b200 as kmb
    out = subprocess.check_output(["nm", "-D", "--defined-only", kmb.LIB_PATH]).decode()
    exported = set(re.findall(r" T (km_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(kmb.LIB_PATH)
    for f in declared_functions():
        assert hasattr(lib, f)


def test_binding_names_match_header():
    from paper_2412_02244_b200 import km
    for f in declared_functions():
        assert f in km.EXPORTED, f


def test_max_k():
    import paper_2412_02244_b200 as kmb
    assert kmb.km_max_k(1) == 0 and kmb.km_max_k(257) == 0
    assert kmb.km_max_k(4) == kmb.km_max_k(100) == kmb.km_max_k(128) == 1 << 20   # high-d variant (padded widths)
    assert kmb.km_max_k(3) >= 10_000 and kmb.km_max_k(2) >= 10_000
    assert kmb.km_max_k(2) % 4 == 0


def test_validation_before_any_cuda_call():
    from paper_2412_02244_b200 import km
    lib = km._lib
    h = ctypes.c_void_p()
    V = ctypes.c_void_p
    assert lib.km_create(None, 10, 2, 2, None) == km.KM_E_INVALID
    assert lib.km_create(ctypes.byref(h), 0, 2, 1, None) == km.KM_E_INVALID       # n < 1
    assert lib.km_create(ctypes.byref(h), 10, 2, 0, None) == km.KM_E_INVALID      # k < 1
    assert lib.km_create(ctypes.byref(h), 10, 2, 11, None) == km.KM_E_INVALID     # k > n
    assert lib.km_create(ctypes.byref(h), 10, 257, 2, None) == km.KM_E_UNSUPPORTED  # d > 256
    assert lib.km_create(ctypes.byref(h), 10, 1, 2, None) == km.KM_E_UNSUPPORTED
    assert lib.km_create(ctypes.byref(h), 10**6, 3, km.km_max_k(3) + 4, None) == km.KM_E_UNSUPPORTED
    assert h.value is None
    sse = ctypes.c_double()
    buf = (ctypes.c_float * 64)()
    lab = (ctypes.c_int32 * 16)()
    assert lib.km_run(None, 16, 2, 2, buf, 3, -1.0, buf, lab, ctypes.byref(sse)) == km.KM_E_INVALID
    assert lib.km_run(buf, 16, 2, 2, buf, 0, -1.0, buf, lab, ctypes.byref(sse)) == km.KM_E_INVALID  # max_iter < 1
    assert lib.km_assign(None, buf, buf, lab, None) == km.KM_E_INVALID
    assert lib.km_update(None, buf, lab, buf, buf, None, None) == km.KM_E_INVALID
    assert lib.km_run_ctx(None, buf, buf, 3, -1.0, buf, lab, ctypes.byref(sse), None, None) == km.KM_E_INVALID
    assert lib.km_destroy(None) == km.KM_OK
    assert lib.km_timing_enable(None, 1) == km.KM_E_INVALID


def test_no_device_is_a_cuda_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_02244_b200 import km
    h = ctypes.c_void_p()
    rc = km._lib.km_create(ctypes.byref(h), 100, 2, 4, None)
    assert rc == km.KM_E_CUDA and h.value is None


def test_strerror():
    from paper_2412_02244_b200 import km
    for c in (0, -1, -2, -3, -4, -5, -99):
        assert isinstance(km._lib.km_strerror(c), bytes)


def test_product_path_does_not_touch_oracle():
    """The product (package + CUDA sources) never imports/links/calls oracle/."""
    pkg = os.path.join(ROOT, "paper_2412_02244_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "liboracle" not in s and "lloyd_oracle" not in s, f
