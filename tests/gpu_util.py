"""Shared helpers for the GPU parity tests (test infrastructure)."""
import numpy as np
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import modulora as M


def qmatrix(words, rows, cols, bits, group, scales, zeros) -> M.QuantizedMatrix:
    return M.QuantizedMatrix(rows=int(rows), cols=int(cols), bits=int(bits), group_size=int(group),
                             codes=M.PackedCodes(bits=int(bits), count=int(rows) * int(cols),
                                                 words=np.asarray(words, np.uint32)),
                             scales=np.asarray(scales, np.float32),
                             zeros=np.asarray(zeros, np.float32))


def random_quantized(rows, cols, bits, group, seed, std=0.02):
    """W ~ N(0, std^2) from the reference Rng, RTN-quantized by the oracle
    (quantize.cpp:163-184) -> (QuantizedMatrix, words, scales, zeros)."""
    w = orc.gaussian(seed, rows, cols, 0.0, std)
    words, scales, zeros = orc.quantize_rtn(w, bits, group)
    g = cols if group == 0 else group
    return qmatrix(words, rows, cols, bits, g, scales, zeros), words, scales, zeros


def to_bf16_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()


def f64(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def deq_bf16_f64(words, rows, cols, bits, group, scales, zeros) -> np.ndarray:
    """Ŵ as the tensor cores see it: bf16(RN_f32(oracle f64)), as f64."""
    return orc.bf16_round(orc.dequantize_f32(words, rows, cols, bits, group, scales, zeros))


# ----------------------------------------------------------------------------- big shapes
def synthetic(rows, cols, bits, group, seed):
    """The bench's own synthetic weights (bench.synthetic_codes: uniform codes,
    RTN-like grids) -> (QuantizedMatrix, words, scales, zeros)."""
    from bench import synthetic_codes
    words, sc, z = synthetic_codes(rows, cols, bits, group, seed)
    return qmatrix(words, rows, cols, bits, group, sc, z), words, sc, z


def sample_rows(m, block=128, seed=0):
    """One seeded token row per `block`-token sub-tile, plus the last row: every
    token tile of every schedule is hit by the sampled-row checks."""
    rng = np.random.default_rng(seed)
    rows = [b + int(rng.integers(0, min(block, m - b))) for b in range(0, m, block)]
    return np.unique(np.array(rows + [m - 1]))


def deq_products(words, rows, cols, bits, group, sc, z, x_rows, g_rows, chunk=2048):
    """Products of sampled activation rows with Ŵ, streamed over row chunks of the
    weights (the oracle dequantizes each chunk; rows must be word-aligned, which
    every BASELINE shape is): returns
      (x·Ŵbfᵀ, x·Ŵᵀ, g·Ŵbf, g·Ŵ) with Ŵbf = bf16(RN_f32(oracle)), Ŵ the f64 oracle."""
    assert (cols * bits) % 32 == 0
    rw = cols * bits // 32
    ng = cols // group
    yb = np.zeros((x_rows.shape[0], rows))
    ye = np.zeros_like(yb)
    db = np.zeros((g_rows.shape[0], cols))
    de = np.zeros_like(db)
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        w_ = words[r0 * rw:r1 * rw]
        s_, z_ = sc[r0 * ng:r1 * ng], z[r0 * ng:r1 * ng]
        wex = orc.dequantize(w_, r1 - r0, cols, bits, group, s_, z_)
        wbf = orc.bf16_round(orc.dequantize_f32(w_, r1 - r0, cols, bits, group, s_, z_))
        yb[:, r0:r1] = x_rows @ wbf.T
        ye[:, r0:r1] = x_rows @ wex.T
        db += g_rows[:, r0:r1] @ wbf
        de += g_rows[:, r0:r1] @ wex
    return yb, ye, db, de


def check_layer_pass(deq, a32, b32, alpha, x64, g64, y, xb, dx, da, db, bias32=None,
                     rows=None, what=""):
    """SURVEY §8(c) bars for one ModuLoRA layer fwd+bwd computed on the device.

    deq(x_rows, g_rows) -> (x·Ŵbfᵀ, x·Ŵᵀ, g·Ŵbf, g·Ŵ) for the sampled rows.
    y, dx: fp32 device results (full); xb, da, db fp32 (full).
      * xb, dA, dB: full, <= 1e-5 / 1e-4 / 1e-4 vs f64 on the same inputs;
      * Y, dX sampled rows: <= 1e-4 vs the GPU recipe in f64 (bf16 Ŵ, bf16(s·xb),
        bf16 A/B), <= 4e-3 vs the exact f64 layer."""
    from tests.conftest import rel_fro
    r = a32.shape[1]
    s = alpha / r
    A, B = a32.astype(np.float64), b32.astype(np.float64)
    xbr = x64 @ B
    dyar = g64 @ A
    e = {}
    e["xb"] = rel_fro(f64(xb), xbr)
    e["dA"] = rel_fro(f64(da), s * (g64.T @ xbr))
    e["dB"] = rel_fro(f64(db), s * (x64.T @ dyar))
    if rows is None:
        rows = sample_rows(x64.shape[0])
    yb, ye, dxb, dxe = deq(x64[rows], g64[rows])
    bias = 0.0 if bias32 is None else bias32.astype(np.float64)[None, :]
    y_recipe = yb + orc.bf16_round(s * xbr[rows]) @ orc.bf16_round(A).T + bias
    y_exact = ye + s * xbr[rows] @ A.T + bias
    e["y_tight"] = rel_fro(f64(y)[rows], y_recipe)
    e["y_loose"] = rel_fro(f64(y)[rows], y_exact)
    if dx is not None:
        dx_recipe = dxb + orc.bf16_round(s * dyar[rows]) @ orc.bf16_round(B).T
        dx_exact = dxe + s * dyar[rows] @ B.T
        e["dx_tight"] = rel_fro(f64(dx)[rows], dx_recipe)
        e["dx_loose"] = rel_fro(f64(dx)[rows], dx_exact)
    bars = {"xb": 1e-5, "dA": 1e-4, "dB": 1e-4, "y_tight": 1e-4, "y_loose": 4e-3,
            "dx_tight": 1e-4, "dx_loose": 4e-3}
    bad = {k: v for k, v in e.items() if not v <= bars[k]}
    assert not bad, f"{what}: {bad} (all: {e})"
    return e
