"""The reference-side drop-in (integration/modulora_gpu.hpp) on the reference's
own tape: oracle/_ref/test_dropin is tests/cpp/test_dropin.cpp compiled against
the reference headers and linked with the reference's own objects (compiled in
place by oracle/Makefile) plus libmlra.so. It re-runs the reference's
acceptance C1 (acceptance.cpp:98-157) and C8 (:421-457) with the GPU
CustomFunction registered on the reference Tape (lowprec_linear.hpp:96-112,
autodiff.hpp:77-89), and the whole layer as one GPU record. The binary is
built here (where /root/reference exists) and travels to the GPU box.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")
REF = "/root/reference/proj/src/lora.cpp"


def _binary():
    if not os.path.exists(BIN) and os.path.exists(REF):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True)
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_dropin not built (needs the reference sources at build time)")
    return BIN


def test_dropin_links_reference_objects_and_libmlra():
    b = _binary()
    out = subprocess.run(["ldd", b], capture_output=True, text=True).stdout
    assert "libmlra.so" in out and "not found" not in out.split("libmlra.so")[1].splitlines()[0]
    syms = subprocess.run(["nm", "-C", b], capture_output=True, text=True).stdout
    # the reference's own tape and layer code are linked in, not re-implemented
    assert "modulora::Tape::backward_from" in syms
    assert "modulora::layer_forward" in syms and "modulora::lp_forward" in syms


@pytest.mark.gpu
def test_reference_acceptance_on_the_gpu_function():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == 4 and all(l.startswith("[PASS]") for l in lines), r.stdout
