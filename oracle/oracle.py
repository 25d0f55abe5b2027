"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by ``oracle/Makefile``:

* ``liboracle.so`` — the plain-C restatement of the reference hot path
  (``oracle/mlra_oracle.c``; every function cites reference file:line). This is
  the parity checker used by ``tests/``, ``__graft_entry__.smoke()`` and the
  ``cpu_baseline`` leg of ``bench.py``.
* ``_ref/libmlra_ref.so`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` plus ``oracle/ref_driver.cpp``. It pins the
  restatement (golden fixtures) and is the CPU baseline of ``bench.py
  --impl reference``. Optional: absent when the reference could not be built.

Nothing in the product package (``paper_2309_16119_b200``) imports this file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64 = C.c_uint64
_int = C.c_int


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class _Lib:
    _lib = None

    @classmethod
    def get(cls) -> C.CDLL:
        if cls._lib is None:
            lib = _load(os.path.join(HERE, "liboracle.so"))
            lib.orc_mix_seed.restype = _u64
            lib.orc_mix_seed.argtypes = [_u64, _u64]
            lib.orc_gaussian_fill.argtypes = [_u64, _f64p, _u64, C.c_double, C.c_double]
            lib.orc_packed_word_count.restype = _u64
            lib.orc_packed_word_count.argtypes = [_u64, _int]
            lib.orc_pack.restype = _int
            lib.orc_pack.argtypes = [_u32p, _u64, _int, _u32p, C.POINTER(_u64)]
            lib.orc_unpack.restype = _int
            lib.orc_unpack.argtypes = [_u32p, _u64, _u64, _int, _u32p]
            lib.orc_validate_packed.restype = _int
            lib.orc_validate_packed.argtypes = [_u32p, _u64, _u64, _int]
            lib.orc_quantize_rtn.restype = _int
            lib.orc_quantize_rtn.argtypes = [_f64p, _u64, _u64, _int, _u64, _u32p, _f32p, _f32p]
            lib.orc_validate_qmatrix.restype = _int
            lib.orc_validate_qmatrix.argtypes = [_u64, _u64, _int, _int, _u64, _u64, _u64, _u64, _f32p]
            lib.orc_dequantize.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _f64p]
            lib.orc_dequantize_f32.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _f32p]
            lib.orc_dequantize_row.argtypes = [_u32p, _u64, _int, _u64, _f32p, _f32p, _u64, _f64p]
            lib.orc_matmul.argtypes = [_f64p, _f64p, _u64, _u64, _u64, _f64p]
            lib.orc_lp_forward_dense.argtypes = [_f64p, _u64, _u64, _f64p, _u64, _f64p]
            lib.orc_lp_backward_dense.argtypes = [_f64p, _u64, _u64, _f64p, _u64, _f64p]
            vp = C.c_void_p
            lib.orc_layer_forward_dense.argtypes = [
                _f64p, _u64, _u64, _f64p, _f64p, _u64, C.c_double, vp, _f64p, _u64, _f64p, _f64p]
            lib.orc_layer_backward_dense.argtypes = [
                _f64p, _u64, _u64, _f64p, _f64p, _u64, C.c_double, _f64p, _f64p, _f64p,
                _u64, vp, _f64p, _f64p, vp]
            lib.orc_cb2_dequant_f32.argtypes = [
                np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS"), _u64, _u64, _u64, _f32p,
                _f32p, _f32p]
            lib.orc_adamw_step.restype = _int
            lib.orc_adamw_step.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, _u64,
                                           C.c_double, _u64, _f64p, _f64p, _f64p, _f64p]
            lib.orc_lut_dequant_f32.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _f32p]
            lib.orc_e8p_abs_table.argtypes = [C.c_void_p]
            lib.orc_e8p_abs_table.restype = None
            lib.orc_e8p_dequant_f32.argtypes = [
                np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS"), _u64, _u64, _u64, _f32p,
                _f32p]
            lib.orc_e8p_dequant_f32.restype = None
            cls._lib = lib
        return cls._lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --- rng.hpp ---------------------------------------------------------------
def mix_seed(seed: int, salt: int) -> int:
    return int(_Lib.get().orc_mix_seed(seed, salt))


def gaussian(seed: int, rows: int, cols: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
    """DenseMatrix::gaussian(rows, cols, Rng(seed), mean, std) (matrix.cpp:62-67)."""
    out = np.empty(rows * cols, np.float64)
    _Lib.get().orc_gaussian_fill(seed, out, rows * cols, mean, std)
    return out.reshape(rows, cols)


# --- bitpack.cpp -------------------------------------------------------------
def packed_word_count(count: int, bits: int) -> int:
    return int(_Lib.get().orc_packed_word_count(count, bits))


def pack(codes, bits: int) -> np.ndarray:
    codes = _c(np.asarray(codes).ravel(), np.uint32)
    n = codes.size
    words = np.zeros(max(packed_word_count(n, bits), 1), np.uint32)
    bad = _u64(0)
    st = _Lib.get().orc_pack(codes, n, bits, words, C.byref(bad))
    if st == -1:
        raise ValueError(f"ConfigError: unsupported bit width {bits}")
    if st == -2:
        raise IndexError(f"RangeError: code at index {bad.value} exceeds {bits}-bit range")
    return words[: packed_word_count(n, bits)]


def unpack(words, count: int, bits: int) -> np.ndarray:
    words = _c(words, np.uint32)
    out = np.zeros(max(count, 1), np.uint32)
    w = words if words.size else np.zeros(1, np.uint32)
    st = _Lib.get().orc_unpack(w, words.size, count, bits, out)
    if st == -1:
        raise ValueError("ConfigError")
    if st == -3:
        raise RuntimeError("FormatError: corrupted packed container")
    return out[:count]


# --- quantize.cpp ------------------------------------------------------------
def quantize_rtn(w: np.ndarray, bits: int, group: int = 0):
    """quantize_rtn (quantize.cpp:163-184) -> (words u32, scales f32, zeros f32)."""
    w = _c(w, np.float64)
    rows, cols = w.shape
    g = cols if group == 0 else group
    ng = rows * (cols // g) if g and cols % g == 0 else 1
    words = np.zeros(max(packed_word_count(rows * cols, bits), 1), np.uint32)
    scales = np.zeros(ng, np.float32)
    zeros = np.zeros(ng, np.float32)
    st = _Lib.get().orc_quantize_rtn(w, rows, cols, bits, group, words, scales, zeros)
    if st:
        raise ValueError(f"quantize_rtn failed: status {st}")
    return words[: packed_word_count(rows * cols, bits)], scales, zeros


def dequantize(words, rows, cols, bits, group, scales, zeros) -> np.ndarray:
    """dequantize (quantize.cpp:117-137), f64."""
    out = np.empty(rows * cols, np.float64)
    _Lib.get().orc_dequantize(_c(words, np.uint32), rows, cols, bits, group,
                              _c(scales, np.float32), _c(zeros, np.float32), out)
    return out.reshape(rows, cols)


def dequantize_f32(words, rows, cols, bits, group, scales, zeros) -> np.ndarray:
    """The materialize() contract: (float)dequantize(...) element-wise."""
    out = np.empty(rows * cols, np.float32)
    _Lib.get().orc_dequantize_f32(_c(words, np.uint32), rows, cols, bits, group,
                                  _c(scales, np.float32), _c(zeros, np.float32), out)
    return out.reshape(rows, cols)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    nan = ((u & 0x7F800000) == 0x7F800000) & ((u & 0x007FFFFF) != 0)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(h, np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Values rounded to bf16 (RN-even), returned as f64."""
    return bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32))).astype(np.float64)


# --- lowprec_linear.cpp / lora.cpp ------------------------------------------
def lp_forward(w: np.ndarray, x: np.ndarray) -> np.ndarray:
    """lp_forward (lowprec_linear.cpp:150-196) given the f64 dequantized W."""
    w = _c(w, np.float64)
    x = _c(x, np.float64)
    out = np.empty((x.shape[0], w.shape[0]), np.float64)
    _Lib.get().orc_lp_forward_dense(w, w.shape[0], w.shape[1], x, x.shape[0], out)
    return out


def lp_backward(w: np.ndarray, g: np.ndarray) -> np.ndarray:
    """lp_backward (lowprec_linear.cpp:198-247) given the f64 dequantized W."""
    w = _c(w, np.float64)
    g = _c(g, np.float64)
    out = np.empty((g.shape[0], w.shape[1]), np.float64)
    _Lib.get().orc_lp_backward_dense(w, w.shape[0], w.shape[1], g, g.shape[0], out)
    return out


def layer_forward(w, a, b, alpha, bias, x):
    """layer_forward (lora.cpp:52-72) -> (y, xb). a: [d_out×r], b: [d_in×r]."""
    w = _c(w, np.float64)
    a = _c(a, np.float64)
    b = _c(b, np.float64)
    x = _c(x, np.float64)
    d_out, d_in = w.shape
    r = a.shape[1]
    m = x.shape[0]
    bias_c = None if bias is None else _c(bias, np.float64).ravel()
    y = np.empty((m, d_out), np.float64)
    xb = np.empty((m, r), np.float64)
    _Lib.get().orc_layer_forward_dense(w, d_out, d_in, a, b, r, float(alpha) / r,
                                       _ptr(bias_c), x, m, y, xb)
    return y, xb


def layer_backward(w, a, b, alpha, x, xb, g, need_dx=True, need_dbias=False):
    """Tape replay of layer_forward's records (autodiff.cpp:101-193)."""
    w = _c(w, np.float64)
    a = _c(a, np.float64)
    b = _c(b, np.float64)
    x = _c(x, np.float64)
    xb = _c(xb, np.float64)
    g = _c(g, np.float64)
    d_out, d_in = w.shape
    r = a.shape[1]
    m = x.shape[0]
    dx = np.empty((m, d_in), np.float64) if need_dx else None
    da = np.empty((d_out, r), np.float64)
    db = np.empty((d_in, r), np.float64)
    dbias = np.empty(d_out, np.float64) if need_dbias else None
    _Lib.get().orc_layer_backward_dense(w, d_out, d_in, a, b, r, float(alpha) / r, x, xb,
                                        g, m, _ptr(dx), da, db, _ptr(dbias))
    return dx, da, db, dbias


# --- the unmodified reference (optional) ------------------------------------
class Ref:
    """The reference library itself (oracle/_ref/libmlra_ref.so)."""

    path = os.path.join(HERE, "_ref", "libmlra_ref.so")
    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.path)

    @classmethod
    def get(cls) -> C.CDLL:
        if cls._lib is None:
            lib = C.CDLL(cls.path)
            vp = C.c_void_p
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_gaussian.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double, _f64p]
            lib.ref_mix_seed.restype = _u64
            lib.ref_mix_seed.argtypes = [_u64, _u64]
            lib.ref_random_codes.argtypes = [_u64, _int, _u64, _u32p]
            lib.ref_packed_word_count.restype = _u64
            lib.ref_packed_word_count.argtypes = [_u64, _int]
            lib.ref_pack.argtypes = [_u32p, _u64, _int, _u32p]
            lib.ref_unpack.argtypes = [_u32p, _u64, _u64, _int, _u32p]
            lib.ref_quantize_rtn.argtypes = [_f64p, _u64, _u64, _int, _u64, _u32p, _f32p, _f32p]
            lib.ref_quantize_optq.argtypes = [_f64p, _f64p, _u64, _u64, _u64, _int, _u64, C.c_double,
                                              _u32p, _f32p, _f32p]
            lib.ref_optq_workspace.argtypes = [_f64p, _u64, _u64, C.c_double, _f64p, _f64p]
            lib.ref_validate.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p]
            lib.ref_dequantize.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _f64p]
            lib.ref_lp_forward.argtypes = [_u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _int,
                                           _f64p, _u64, _f64p]
            lib.ref_lp_backward.argtypes = lib.ref_lp_forward.argtypes
            lib.ref_init_adapter_b.argtypes = [_u64, _u64, _u64, C.c_double, _u64, _f64p]
            lib.ref_layer_fwd_bwd.argtypes = [
                _u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _int, _f64p, _f64p, _u64,
                C.c_double, vp, _f64p, _u64, _f64p, _f64p, vp, _f64p, _f64p, vp]
            lib.ref_bench_layer.argtypes = [
                _u32p, _u64, _u64, _int, _u64, _f32p, _f32p, _int, _u64, C.c_double, _u64,
                _int, _u64, C.POINTER(C.c_double)]
            lib.ref_adamw_run.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, _u64,
                                          np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                          _f64p, _f64p, _u64, _f64p, C.POINTER(_u64)]
            lib.ref_adamw_run.restype = _int
            lib.ref_parity_loss_grads.argtypes = [C.c_char_p, _f64p,
                                                  np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                                  _u64, _u64, _u64, C.POINTER(C.c_double), _f64p, _u64]
            lib.ref_parity_loss_grads.restype = _int
            cls._lib = lib
        return cls._lib

    @classmethod
    def adamw_run(cls, sizes, values, grads, lrs, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0):
        """The reference AdamW over len(lrs) steps; returns (rc, values, bad_step)."""
        vals = np.ascontiguousarray(values, np.float64).copy()
        bad = _u64(0)
        rc = cls.get().ref_adamw_run(beta1, beta2, eps, wd, len(sizes),
                                     np.asarray(sizes, np.uint64), vals,
                                     np.ascontiguousarray(grads, np.float64).ravel(), len(lrs),
                                     np.ascontiguousarray(lrs, np.float64), C.byref(bad))
        return rc, vals, int(bad.value)

    @classmethod
    def parity_loss_grads(cls, path: str, xs, labels, n_grads: int):
        """The reference's parity-transformer model_loss + tape backward on the
        checkpoint at ``path``: (loss, flat trainable-param grads)."""
        xs = np.ascontiguousarray(xs, np.float64)
        n, seq, d = xs.shape
        g = np.empty(n_grads, np.float64)
        loss = C.c_double()
        cls._chk(cls.get().ref_parity_loss_grads(path.encode(), xs.ravel(),
                                                 np.ascontiguousarray(labels, np.int32), n, seq, d,
                                                 C.byref(loss), g, n_grads))
        return loss.value, g

    @classmethod
    def _chk(cls, st):
        if st:
            raise RuntimeError(f"reference error {st}: {cls.get().ref_last_error().decode()}")

    @classmethod
    def gaussian(cls, seed, rows, cols, mean=0.0, std=1.0):
        out = np.empty(rows * cols, np.float64)
        cls.get().ref_gaussian(seed, rows, cols, mean, std, out)
        return out.reshape(rows, cols)

    @classmethod
    def random_codes(cls, n, bits, seed):
        out = np.zeros(max(n, 1), np.uint32)
        cls.get().ref_random_codes(n, bits, seed, out)
        return out[:n]

    @classmethod
    def pack(cls, codes, bits):
        codes = _c(np.asarray(codes).ravel(), np.uint32)
        nw = int(cls.get().ref_packed_word_count(codes.size, bits))
        words = np.zeros(max(nw, 1), np.uint32)
        cls._chk(cls.get().ref_pack(codes if codes.size else np.zeros(1, np.uint32),
                                    codes.size, bits, words))
        return words[:nw]

    @classmethod
    def quantize_rtn(cls, w, bits, group=0):
        w = _c(w, np.float64)
        rows, cols = w.shape
        g = cols if group == 0 else group
        nw = int(cls.get().ref_packed_word_count(rows * cols, bits))
        words = np.zeros(max(nw, 1), np.uint32)
        scales = np.zeros(rows * (cols // g), np.float32)
        zeros = np.zeros(rows * (cols // g), np.float32)
        cls._chk(cls.get().ref_quantize_rtn(w, rows, cols, bits, group, words, scales, zeros))
        return words[:nw], scales, zeros

    @classmethod
    def quantize_optq(cls, w, calib, bits, group=0, damping=0.01):
        w = _c(w, np.float64)
        calib = _c(calib, np.float64)
        rows, cols = w.shape
        g = cols if group == 0 else group
        nw = int(cls.get().ref_packed_word_count(rows * cols, bits))
        words = np.zeros(max(nw, 1), np.uint32)
        scales = np.zeros(rows * (cols // g), np.float32)
        zeros = np.zeros(rows * (cols // g), np.float32)
        cls._chk(cls.get().ref_quantize_optq(w, calib, rows, cols, calib.shape[0], bits, group,
                                             damping, words, scales, zeros))
        return words[:nw], scales, zeros

    @classmethod
    def optq_workspace(cls, calib, damping=0.01):
        calib = _c(calib, np.float64)
        m, n = calib.shape
        h = np.zeros((n, n), np.float64)
        u = np.zeros((n, n), np.float64)
        cls._chk(cls.get().ref_optq_workspace(calib, m, n, damping, h, u))
        return h, u

    @classmethod
    def dequantize(cls, words, rows, cols, bits, group, scales, zeros):
        out = np.empty(rows * cols, np.float64)
        cls._chk(cls.get().ref_dequantize(_c(words, np.uint32), rows, cols, bits, group,
                                          _c(scales, np.float32), _c(zeros, np.float32), out))
        return out.reshape(rows, cols)

    @classmethod
    def layer_fwd_bwd(cls, words, rows, cols, bits, group, scales, zeros, a, b, alpha, bias,
                      x, g, need_dx=True, need_dbias=False, strategy=0):
        m = x.shape[0]
        r = a.shape[1]
        y = np.empty((m, rows), np.float64)
        dx = np.empty((m, cols), np.float64) if need_dx else None
        da = np.empty((rows, r), np.float64)
        db = np.empty((cols, r), np.float64)
        dbias = np.empty(rows, np.float64) if need_dbias else None
        bias_c = None if bias is None else _c(bias, np.float64).ravel()
        cls._chk(cls.get().ref_layer_fwd_bwd(
            _c(words, np.uint32), rows, cols, bits, group, _c(scales, np.float32),
            _c(zeros, np.float32), strategy, _c(a, np.float64), _c(b, np.float64), r,
            float(alpha), _ptr(bias_c), _c(x, np.float64), m, _c(g, np.float64), y,
            _ptr(dx), da, db, _ptr(dbias)))
        return y, dx, da, db, dbias

    @classmethod
    def bench_layer(cls, words, rows, cols, bits, group, scales, zeros, rank, alpha,
                    m_per_thread, threads, seed=1, strategy=1):
        secs = C.c_double(0.0)
        cls._chk(cls.get().ref_bench_layer(
            _c(words, np.uint32), rows, cols, bits, group, _c(scales, np.float32),
            _c(zeros, np.float32), strategy, rank, float(alpha), m_per_thread, threads, seed,
            C.byref(secs)))
        return secs.value


# --- cb2 plugin decode law (include/mlra.h mlra_cb2_create) ------------------
def cb2_dequantize_f32(codes, rows: int, cols: int, group: int, codebook, scales) -> np.ndarray:
    """orc_cb2_dequant_f32: the f32 image of the cb2 codebook plugin."""
    out = np.empty(rows * cols, np.float32)
    _Lib.get().orc_cb2_dequant_f32(_c(codes, np.uint16).ravel(), rows, cols, group,
                                   _c(codebook, np.float32).ravel(),
                                   _c(scales, np.float32).ravel(), out)
    return out.reshape(rows, cols)


# --- e8p plugin decode law (include/mlra.h mlra_e8p_create) -------------------
def e8p_abs_table() -> np.ndarray:
    """orc_e8p_abs_table: the 256 E8P abs patterns, 2|a| as int32 [256, 8]."""
    t = np.empty(256 * 8, np.int32)
    _Lib.get().orc_e8p_abs_table(t.ctypes.data_as(C.c_void_p))
    return t.reshape(256, 8)


def e8p_dequantize_f32(codes, rows: int, cols: int, group: int, scales) -> np.ndarray:
    """orc_e8p_dequant_f32: RN_f32(s * (sign * |a| +- 1/4)) per entry."""
    out = np.empty(rows * cols, np.float32)
    _Lib.get().orc_e8p_dequant_f32(_c(codes, np.uint16).ravel(), rows, cols, group,
                                   _c(scales, np.float32).ravel(), out)
    return out.reshape(rows, cols)


# --- train.cpp AdamW ------------------------------------------------------------
def adamw_step(params, ms, vs, grads, step_index: int, lr: float, beta1=0.9, beta2=0.999,
               eps=1e-8, weight_decay=0.0) -> int:
    """AdamW::step (train.cpp:81-134) over a list of f64 arrays, updated in
    place in order. Returns the index of the first parameter whose gradient is
    non-finite (it and the rest untouched), or len(params)."""
    for i, (p, m, v, g) in enumerate(zip(params, ms, vs, grads)):
        rc = _Lib.get().orc_adamw_step(beta1, beta2, eps, weight_decay, step_index, lr, p.size,
                                       p.reshape(-1), m.reshape(-1), v.reshape(-1),
                                       _c(g, np.float64).reshape(-1))
        if rc:
            return i
    return len(params)


# --- lut plugin decode law (include/mlra.h mlra_lut_create) -------------------
def lut_dequantize_f32(words, rows: int, cols: int, bits: int, group: int, lut, scales) -> np.ndarray:
    """orc_lut_dequant_f32: RN_f32(s * lut[c]) per entry."""
    out = np.empty(rows * cols, np.float32)
    _Lib.get().orc_lut_dequant_f32(_c(words, np.uint32).ravel(), rows, cols, bits, group,
                                   _c(lut, np.float32).ravel(), _c(scales, np.float32).ravel(), out)
    return out.reshape(rows, cols)
