"""OPTQ on the device: OptqQuantizer / mlra_quantize_optq and
mlra_optq_workspace against the reference's own quantize_optq and
build_optq_workspace (quantize.cpp:186-255, linalg.cpp:13-71), bit for bit.

tests/golden/optq.npz holds the reference's outputs (words, scales, zeros;
the Hessian and inverse-Cholesky factor for the small cases) on seeded inputs
that tests/golden/make_golden.py regenerates (the fixture pins their digest).
"""
import importlib.util
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import modulora as M

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _mg():
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLDEN, "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


MG = _mg()
Z = np.load(os.path.join(GOLDEN, "optq.npz"))
CASES = list(range(len(MG.OPTQ_CASES)))


def _case(ci):
    rows, cols, m, bits, group, damp = MG.OPTQ_CASES[ci]
    w, x = MG.optq_inputs(ci)
    assert MG.input_digest(w, x) == int(Z[f"c{ci}_digest"][0]), "seeded inputs drifted"
    return rows, cols, m, bits, group, damp, w, x


# ----------------------------------------------------------------------------- CPU
@pytest.mark.parametrize("ci", CASES)
def test_fixture_matches_live_reference(ci):
    if not orc.Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    rows, cols, m, bits, group, damp, w, x = _case(ci)
    words, scales, zeros = orc.Ref.quantize_optq(w, x, bits, group, damp)
    assert np.array_equal(words, Z[f"c{ci}_words"])
    assert np.array_equal(scales, Z[f"c{ci}_scales"]) and np.array_equal(zeros, Z[f"c{ci}_zeros"])


def test_optq_beats_rtn_on_the_proxy_loss():
    # the reference's own claim (the sweep minimises ||X Wᵀ - X Ŵᵀ||²): pinned
    # on the fixture, so the GPU parity below inherits it
    for ci in CASES:
        rows, cols, m, bits, group, damp, w, x = _case(ci)
        g = cols if group == 0 else group
        wo = orc.dequantize(Z[f"c{ci}_words"], rows, cols, bits, g, Z[f"c{ci}_scales"], Z[f"c{ci}_zeros"])
        rw, rs, rz = orc.quantize_rtn(w, bits, group)
        wr = orc.dequantize(rw, rows, cols, bits, g, rs, rz)
        lo = np.linalg.norm(x @ (w - wo).T) ** 2
        lr = np.linalg.norm(x @ (w - wr).T) ** 2
        assert lo <= lr * 1.0001, (ci, lo, lr)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("ci", [c for c in CASES if f"c{c}_h" in Z.files])
def test_optq_workspace_bit_exact(ci):
    rows, cols, m, bits, group, damp, w, x = _case(ci)
    h, u = M.optq_workspace(x, damp)
    assert np.array_equal(h.cpu().numpy(), Z[f"c{ci}_h"])
    assert np.array_equal(u.cpu().numpy(), Z[f"c{ci}_u"])


@pytest.mark.gpu
@pytest.mark.parametrize("ci", CASES)
def test_optq_quantize_bit_exact(ci):
    rows, cols, m, bits, group, damp, w, x = _case(ci)
    q = M.OptqQuantizer(damp).quantize(w, x, bits, group)
    assert np.array_equal(q.scales, Z[f"c{ci}_scales"])
    assert np.array_equal(q.zeros, Z[f"c{ci}_zeros"])
    assert np.array_equal(q.codes.words, Z[f"c{ci}_words"])
    # and it uploads / dequantizes like any QuantizedMatrix
    dq = M.DeviceQuantizedMatrix(q)
    want = orc.dequantize_f32(q.codes.words, rows, cols, bits, q.group_size, q.scales, q.zeros)
    assert np.array_equal(M.dequantize(dq, torch.float32).cpu().numpy(), want)


@pytest.mark.gpu
def test_optq_errors():
    qz = M.OptqQuantizer()
    w = np.random.default_rng(1).normal(0, 0.02, (8, 16))
    x = np.random.default_rng(2).normal(0, 1, (32, 16))
    with pytest.raises(MlraError) as e:
        qz.quantize(np.zeros((0, 16)), x, 4, 8)
    assert e.value.status == 2
    with pytest.raises(MlraError) as e:
        qz.quantize(w, x, 5, 8)
    assert e.value.status == 3
    with pytest.raises(MlraError) as e:
        qz.quantize(w, x, 4, 7)
    assert e.value.status == 3
    with pytest.raises(MlraError) as e:
        M.OptqQuantizer(-1.0).quantize(w, x, 4, 8)
    assert e.value.status == 3
    with pytest.raises(MlraError) as e:
        qz.quantize(w, x[:, :12], 4, 8)
    assert e.value.status == 2
    # an all-zero calibration column without damping: H is singular (exact 0 pivot)
    xs = x.copy()
    xs[:, 5] = 0.0
    with pytest.raises(MlraError) as e:
        M.OptqQuantizer(0.0).quantize(w, xs, 4, 8)
    assert e.value.status == 6 and "not invertible" in str(e.value)
    if orc.Ref.available():
        with pytest.raises(RuntimeError):
            orc.Ref.quantize_optq(w, xs, 4, 8, 0.0)
    # damping rescues it, as in the reference
    M.OptqQuantizer(0.01).quantize(w, xs, 4, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,m,bits,group", [(300, 640, 900, 4, 128), (96, 1024, 1500, 3, 64)])
def test_optq_bit_exact_vs_live_reference_medium(rows, cols, m, bits, group):
    # beyond the fixtures: the compiled reference (oracle/_ref, travels with the
    # repo) on medium shapes — several Cholesky panels, many sweep blocks
    if not orc.Ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(rows + cols)
    w = rng.normal(0.0, 0.02, (rows, cols))
    x = rng.normal(0.0, 1.0, (m, cols))
    x[1:] = 0.5 * x[:-1] + 0.85 * x[1:]
    words, scales, zeros = orc.Ref.quantize_optq(w, x, bits, group, 0.01)
    q = M.OptqQuantizer(0.01).quantize(w, x, bits, group)
    assert np.array_equal(q.scales, scales) and np.array_equal(q.zeros, zeros)
    assert np.array_equal(q.codes.words, words)
    h, u = orc.Ref.optq_workspace(x, 0.01)
    hd, ud = M.optq_workspace(x, 0.01)
    assert np.array_equal(hd.cpu().numpy(), h) and np.array_equal(ud.cpu().numpy(), u)
