"""CPU tests of the C-ABI boundary: the library loads, exports exactly what
include/mlra.h declares, and validates uploads with the reference's error
taxonomy before touching a device (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2309_16119_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mlra.h")).read()
    return sorted(set(re.findall(r"MLRA_API\s+[\w\s\*]+?\b(mlra_\w+)\s*\(", src)))


def test_header_matches_binding_list():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mlra_\w+)", out))
    missing = set(_declared()) - exported
    assert not missing, missing
    L = _lib.lib()
    for name in _declared():
        assert getattr(L, name) is not None


def test_packed_word_count_matches_reference():
    L = _lib.lib()
    for n, b in [(4, 2), (11, 3), (32, 8), (0, 4), (16, 2), (17, 2), (4096 * 4096, 3)]:
        assert L.mlra_packed_word_count(n, b) == orc.packed_word_count(n, b)


def _create(rows, cols, bits, group, words, count, scales, zeros):
    L = _lib.lib()
    h = C.c_void_p()
    words = np.ascontiguousarray(words, np.uint32) if len(words) else np.zeros(1, np.uint32)
    scales = np.ascontiguousarray(scales, np.float32)
    zeros = np.ascontiguousarray(zeros, np.float32)
    st = L.mlra_qweight_create(rows, cols, bits, group, words.ctypes.data,
                               len(words), count, scales.ctypes.data, zeros.ctypes.data,
                               len(scales), None, C.byref(h))
    if st == 0:
        L.mlra_qweight_destroy(h)
    return st, L.mlra_last_error().decode()


def test_upload_validation_taxonomy():
    # quantize.cpp:82-115 and bitpack.cpp:37-60, same exception classes
    w, s, z = orc.quantize_rtn(orc.gaussian(1, 4, 8), 4, 4)
    assert _create(4, 8, 5, 4, w, 32, s, z)[0] == 3          # ConfigError: bits
    assert _create(4, 8, 4, 3, w, 32, s, z)[0] == 3          # ConfigError: group
    assert _create(4, 8, 4, 4, w, 31, s, z)[0] == 7          # FormatError: code count
    assert _create(4, 8, 4, 4, w, 32, s[:-1], z[:-1])[0] == 7  # FormatError: grid count
    bad = s.copy()
    bad[2] = 0.0
    assert _create(4, 8, 4, 4, w, 32, bad, z)[0] == 6        # NumericError: scale <= 0
    assert _create(4, 8, 4, 4, w[:-1], 32, s, z)[0] == 7     # FormatError: word count
    w3, s3, z3 = orc.quantize_rtn(orc.gaussian(2, 1, 11), 3, 11)
    tr = w3.copy()
    tr[-1] |= 0x80000000
    st, msg = _create(1, 11, 3, 11, tr, 11, s3, z3)
    assert st == 7 and "trailing" in msg                     # FormatError: trailing bits


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback():
    w, s, z = orc.quantize_rtn(orc.gaussian(1, 4, 8), 4, 4)
    st, msg = _create(4, 8, 4, 4, w, 32, s, z)
    assert st == 9, msg  # MLRA_ERR_UNSUPPORTED: valid input, but no sm_100 device
    assert _lib.lib().mlra_device_check() == 9


def test_host_rng_matches_reference_stream():
    # rng.hpp:15-57 restated in libmlra (init_adapter's stream): bit-identical to the
    # golden fixtures made by the reference and to the oracle
    import ctypes as C
    from tests.conftest import load_golden
    L = _lib.lib()
    g = load_golden("rng.npz")
    out = np.empty(15, np.float64)
    L.mlra_gaussian_fill(7, out.ctypes.data_as(C.c_void_p), 15, 0.0, 1.0)
    assert np.array_equal(out.view(np.uint64), g["gaussian_seed7"].ravel().view(np.uint64))
    out = np.empty(16, np.float64)
    L.mlra_gaussian_fill(8, out.ctypes.data_as(C.c_void_p), 16, 0.5, 0.02)
    assert np.array_equal(out.view(np.uint64), g["gaussian_seed8_scaled"].ravel().view(np.uint64))
    assert L.mlra_mix_seed(11, 0xADA9) == int(g["mix_seed_11_ada9"][0])
    big = np.empty(4096 * 16, np.float64)
    L.mlra_gaussian_fill(123, big.ctypes.data_as(C.c_void_p), big.size, 0.0, 0.02)
    assert np.array_equal(big.view(np.uint64), orc.gaussian(123, 4096, 16, 0.0, 0.02).ravel().view(np.uint64))
    if orc.Ref.available():
        b = np.empty(300 * 8, np.float64)
        assert orc.Ref.get().ref_init_adapter_b(300, 200, 8, 16.0, 99, b) == 0
        mine = np.empty(300 * 8, np.float64)
        L.mlra_gaussian_fill(99, mine.ctypes.data_as(C.c_void_p), mine.size, 0.0, 0.02)
        assert np.array_equal(mine.view(np.uint64), b.view(np.uint64))
