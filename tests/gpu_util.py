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
