"""Host-side mirror of the reference's hot-path API, on device tensors.

Same names, argument meaning and error behaviour as the reference headers
(quantize.hpp, lowprec_linear.hpp, lora.hpp), re-targeted at libmlra.so:

  reference (CPU, f64)                         here (B200, bf16 operands / fp32 accumulate)
  ------------------------------------------   ---------------------------------------------
  QuantizedMatrix / PackedCodes                QuantizedMatrix / PackedCodes (host containers)
  (upload: none)                               DeviceQuantizedMatrix  -> mlra_qweight_create
  dequantize / dequantize_row                  dequantize / dequantize_row -> mlra_materialize*
  MaterializationStrategy, parse_strategy      same (weight | row | matvec)
  LpLinearContext, lp_forward, lp_backward     same -> mlra_lp_forward / mlra_lp_backward
  LoraAdapter, ModuLoraLayer, make_layer       same (A [d_out x r], B [d_in x r], fp32 masters)
  layer_forward (+ tape backward)              layer_forward / layer_backward -> mlra_lora_*
  grads_of_adapter                             same
  CustomFunction (LpLinearFunction)            ModuLoraLinearFunction (torch.autograd.Function)

Errors raise MlraError whose .kind names the reference exception type.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import MlraError, MlraLora, check, lib


class MaterializationStrategy(enum.IntEnum):
    """lowprec_linear.hpp:29-30."""
    WeightMaterialize = _lib.WEIGHT
    RowMaterialize = _lib.ROW
    QuantizerMatvec = _lib.MATVEC


_NAMES = {"weight": MaterializationStrategy.WeightMaterialize,
          "row": MaterializationStrategy.RowMaterialize,
          "matvec": MaterializationStrategy.QuantizerMatvec}


def parse_strategy(name: str) -> MaterializationStrategy:
    """lowprec_linear.cpp:45-51."""
    if name not in _NAMES:
        raise MlraError(3, f"unknown materialization strategy '{name}' (expected weight, row or matvec)")
    return _NAMES[name]


def strategy_name(s: MaterializationStrategy) -> str:
    return {v: k for k, v in _NAMES.items()}[MaterializationStrategy(s)]


def packed_word_count(count: int, bits: int) -> int:
    """bitpack.cpp:64-66."""
    return int(lib().mlra_packed_word_count(count, bits))


@dataclass
class PackedCodes:
    """bitpack.hpp:17-23."""
    bits: int
    count: int
    words: np.ndarray  # uint32

    def packed_bytes(self) -> int:
        return int(self.words.size) * 4


@dataclass
class QuantizedMatrix:
    """quantize.hpp:29-48 (host container; upload with DeviceQuantizedMatrix)."""
    rows: int
    cols: int
    bits: int
    group_size: int
    codes: PackedCodes
    scales: np.ndarray  # float32 [rows * cols/group]
    zeros: np.ndarray   # float32

    def num_groups(self) -> int:
        return self.cols // self.group_size if self.group_size else 0


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _lib.F32
    if dt == torch.bfloat16:
        return _lib.BF16
    raise MlraError(3, f"unsupported dtype {dt}")


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class DeviceQuantizedMatrix:
    """A frozen QuantizedMatrix resident in HBM (validated on upload exactly as
    QuantizedMatrix::validate, quantize.cpp:82-115). Opaque (plugin-owned)
    formats come from ``Codebook2Quantizer.upload`` / ``opaque``."""

    @classmethod
    def _wrap(cls, h: C.c_void_p, rows: int, cols: int, bits: int, group: int,
              keepalive=None) -> "DeviceQuantizedMatrix":
        self = cls.__new__(cls)
        self._h = h
        self.rows, self.cols, self.bits, self.group_size = rows, cols, bits, group
        self._keepalive = keepalive
        return self

    @classmethod
    def opaque(cls, rows: int, cols: int, bits: int, hook: "QuantizerHook") -> "DeviceQuantizedMatrix":
        """mlra_qweight_create_opaque: a matrix only its plugin can dequantize;
        every strategy materializes it through ``hook``."""
        h = C.c_void_p()
        check(lib().mlra_qweight_create_opaque(rows, cols, bits, C.byref(hook.c_hook()), C.byref(h)))
        return cls._wrap(h, rows, cols, bits, cols, keepalive=hook)

    def __init__(self, q: QuantizedMatrix, stream: Optional[torch.cuda.Stream] = None):
        words = np.ascontiguousarray(q.codes.words, np.uint32)
        scales = np.ascontiguousarray(q.scales, np.float32)
        zeros = np.ascontiguousarray(q.zeros, np.float32)
        if q.codes.bits != q.bits:
            raise MlraError(3, f"QuantizedMatrix: packed bits {q.codes.bits} != {q.bits}")
        h = C.c_void_p()
        dummy = np.zeros(1, np.uint32)
        wp = words if words.size else dummy
        sp = scales if scales.size else dummy.view(np.float32)
        zp = zeros if zeros.size else dummy.view(np.float32)
        check(lib().mlra_qweight_create(
            q.rows, q.cols, q.bits, q.group_size, wp.ctypes.data, words.size, q.codes.count,
            sp.ctypes.data, zp.ctypes.data, scales.size, _stream_ptr(stream), C.byref(h)))
        self._h = h
        self.rows, self.cols, self.bits, self.group_size = q.rows, q.cols, q.bits, q.group_size

    @property
    def handle(self) -> int:
        return self._h.value

    def info(self) -> dict:
        r, c, g, u = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        b, nbytes = C.c_int(), C.c_uint64()
        check(lib().mlra_qweight_info(self._h, C.byref(r), C.byref(c), C.byref(b), C.byref(g),
                                      C.byref(nbytes), C.byref(u)))
        return dict(rows=r.value, cols=c.value, bits=b.value, group_size=g.value,
                    device_bytes=nbytes.value, uncertified_groups=u.value)

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h is not None and h.value and _lib._lib is not None:
                lib().mlra_qweight_destroy(h)
                self._h = C.c_void_p()
        except Exception:  # interpreter shutdown: module globals already torn down
            pass


def dequantize(q: DeviceQuantizedMatrix, dtype: torch.dtype = torch.float32,
               out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """dequantize / dequantize_into (quantize.cpp:117-137) -> device [rows x cols]."""
    if out is None:
        out = torch.empty(q.rows, q.cols, dtype=dtype, device="cuda")
    check(lib().mlra_materialize(q.handle, out.data_ptr(), _dtype_code(out.dtype), out.stride(0),
                                 _stream_ptr(None)))
    return out


def dequantize_tile(q: DeviceQuantizedMatrix, row0: int, nrows: int, col0: int, ncols: int,
                    dtype: torch.dtype = torch.float32, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """mlra_materialize_tile: Ŵ[row0:row0+nrows, col0:col0+ncols] (col0 % 8 == 0)
    — the unit of work of the device dequant hook."""
    if out is None:
        out = torch.empty(nrows, ncols, dtype=dtype, device="cuda")
    check(lib().mlra_materialize_tile(q.handle, row0, nrows, col0, ncols, out.data_ptr(),
                                      _dtype_code(out.dtype), out.stride(0), _stream_ptr(None)))
    return out


def dequantize_row(q: DeviceQuantizedMatrix, row: int, dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """dequantize_row (quantize.cpp:139-161); RangeError past the last row."""
    out = torch.empty(1, q.cols, dtype=dtype, device="cuda")
    check(lib().mlra_materialize_rows(q.handle, row, 1, out.data_ptr(), _dtype_code(dtype),
                                      q.cols, _stream_ptr(None)))
    return out[0]


# --------------------------------------------------------------------------- plugins
class _CudaArray:
    """Zero-copy view of a raw device buffer (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, rows: int, cols: int, ld: int, esize: int):
        self.__cuda_array_interface__ = {
            "data": (ptr, False), "shape": (rows, cols), "strides": (ld * esize, esize),
            "typestr": "<f4" if esize == 4 else "<i2", "version": 2}


class QuantizerHook:
    """The black-box Quantizer plugin (quantize.hpp:91-106) in device form.

    The reference lets a plugin override ``Quantizer::matvec`` /
    ``matvec_transposed`` (quantize.hpp:98-105); lp_forward / lp_backward call
    them under QuantizerMatvec (lowprec_linear.cpp:174-182, 226-235). On the
    GPU the override point is the plugin's dequantization of one tile of Ŵ:
    subclasses implement :meth:`materialize`, writing the tile into ``out`` (a
    bf16 or fp32 CUDA view with the caller's leading dimension) on ``stream``.
    The library then runs its own tcgen05 GEMM over hook-materialized slabs.
    """

    def name(self) -> str:
        return type(self).__name__

    def materialize(self, q: int, row0: int, nrows: int, col0: int, ncols: int,
                    out: torch.Tensor, stream: torch.cuda.Stream) -> None:
        raise NotImplementedError

    def _call(self, _state, q, row0, nrows, col0, ncols, out, dtype, ld, stream):
        try:
            esize = 4 if dtype == _lib.F32 else 2
            view = torch.as_tensor(_CudaArray(out, nrows, ncols, ld, esize), device="cuda")
            if esize == 2:
                view = view.view(torch.bfloat16)
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            self.materialize(q, row0, nrows, col0, ncols, view, st)
            return 0
        except MlraError as e:
            self._error = e
            return e.status
        except Exception as e:  # noqa: BLE001 — reported as a contract failure of the plugin
            self._error = e
            return 5

    def c_hook(self) -> _lib.MlraHook:
        if getattr(self, "_c", None) is None:
            self._fn = _lib.HOOK_FN(self._call)
            self._name = self.name().encode()
            self._c = _lib.MlraHook(self._name, None, self._fn)
        return self._c


class DoublingQuantizer(QuantizerHook):
    """The reference test plugin (test_lowprec.cpp:354-377): the hook returns
    twice the default product, so outputs under QuantizerMatvec double."""

    def materialize(self, q, row0, nrows, col0, ncols, out, stream):
        check(lib().mlra_materialize_tile(q, row0, nrows, col0, ncols, out.data_ptr(),
                                          _dtype_code(out.dtype), out.stride(0), stream.cuda_stream))
        with torch.cuda.stream(stream):
            out.mul_(2)


class RtnQuantizer:
    """The reference's built-in plugin RtnQuantizer (quantize.hpp:108-113):
    round-to-nearest per-(row, group) affine grids. ``quantize`` runs on the
    device (mlra_quantize_rtn) and returns the reference's host QuantizedMatrix
    layout, bit-identical to quantize_rtn((double)w)."""

    def name(self) -> str:
        return "rtn"

    def quantize(self, w, calib=None, bits: int = 4, group_size: int = 0) -> QuantizedMatrix:
        t = torch.as_tensor(w)
        if t.dim() != 2:
            raise MlraError(2, "quantize: expected a 2-D weight matrix")
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        t = t.contiguous().cuda()
        rows, cols = t.shape
        g = cols if group_size == 0 else group_size
        nw = packed_word_count(rows * cols, bits) if rows and cols else 0
        words = torch.empty(max(nw, 1), dtype=torch.int32, device="cuda")
        ng = rows * (cols // g) if g and cols % g == 0 else 0
        scales = torch.empty(max(ng, 1), dtype=torch.float32, device="cuda")
        zeros = torch.empty(max(ng, 1), dtype=torch.float32, device="cuda")
        check(lib().mlra_quantize_rtn(t.data_ptr(), _lib.F64 if t.dtype == torch.float64 else _lib.F32,
                                      rows, cols, bits, group_size, words.data_ptr(),
                                      scales.data_ptr(), zeros.data_ptr(), _stream_ptr(None)))
        wh = words[:nw].cpu().numpy().view(np.uint32).copy()
        return QuantizedMatrix(rows, cols, bits, g, PackedCodes(bits, rows * cols, wh),
                               scales[:ng].cpu().numpy(), zeros[:ng].cpu().numpy())


class OptqQuantizer:
    """The reference's calibration-aware plugin OptqQuantizer (quantize.hpp:115-125):
    H = XᵀX + damping·mean(diag)·I, the upper Cholesky factor of H⁻¹, and the
    error-feeding column sweep (quantize.cpp:186-255) — all on the device
    (mlra_quantize_optq), bit-identical to quantize_optq. Returns the
    reference's host QuantizedMatrix layout (grids as RTN's)."""

    def __init__(self, damping: float = 0.01):
        self.damping = float(damping)

    def name(self) -> str:
        return "optq"

    def quantize(self, w, calib, bits: int = 4, group_size: int = 0) -> QuantizedMatrix:
        t = torch.as_tensor(w)
        if t.dim() != 2:
            raise MlraError(2, "quantize: expected a 2-D weight matrix")
        if calib is None:
            raise MlraError(5, "optq: calibration data required")
        x = torch.as_tensor(calib)
        if x.dim() != 2 or (t.numel() and x.shape[1] != t.shape[1]):
            raise MlraError(2, f"optq: calibration must be [m x {t.shape[1]}], got {tuple(x.shape)}")
        t = t.double().contiguous().cuda()
        x = x.double().contiguous().cuda()
        rows, cols = t.shape
        g = cols if group_size == 0 else group_size
        nw = packed_word_count(rows * cols, bits) if rows and cols else 0
        words = torch.empty(max(nw, 1), dtype=torch.int32, device="cuda")
        ng = rows * (cols // g) if g and cols % g == 0 else 0
        scales = torch.empty(max(ng, 1), dtype=torch.float32, device="cuda")
        zeros = torch.empty(max(ng, 1), dtype=torch.float32, device="cuda")
        check(lib().mlra_quantize_optq(t.data_ptr(), x.data_ptr(), rows, cols, x.shape[0], bits,
                                       group_size, self.damping, words.data_ptr(),
                                       scales.data_ptr(), zeros.data_ptr(), _stream_ptr(None)))
        wh = words[:nw].cpu().numpy().view(np.uint32).copy()
        return QuantizedMatrix(rows, cols, bits, g, PackedCodes(bits, rows * cols, wh),
                               scales[:ng].cpu().numpy(), zeros[:ng].cpu().numpy())


def optq_workspace(calib, damping: float = 0.01):
    """build_optq_workspace (quantize.cpp:186-211) on the device: (hessian,
    inv_chol_upper) as f64 device tensors, bit-identical to the reference."""
    x = torch.as_tensor(calib).double().contiguous().cuda()
    if x.dim() != 2:
        raise MlraError(2, "optq: calibration must be 2-D")
    m, n = x.shape
    h = torch.empty(max(n, 1), max(n, 1), dtype=torch.float64, device="cuda")
    u = torch.empty_like(h)
    check(lib().mlra_optq_workspace(x.data_ptr(), m, n, float(damping), h.data_ptr(), u.data_ptr(),
                                    _stream_ptr(None)))
    return h, u


def default_cb2_codebook() -> np.ndarray:
    """The cb2 plugin's default 256 x 8 magnitude codebook: the 256 shortest
    vectors of {1/2, 3/2, 5/2, 7/2}^8 (a shifted-lattice shell, as in QuIP#'s
    E8-derived codebooks), ordered by squared norm then lexicographically."""
    vals = np.array([0.5, 1.5, 2.5, 3.5])
    idx = np.stack(np.meshgrid(*([np.arange(4)] * 8), indexing="ij"), -1).reshape(-1, 8)
    vecs = vals[idx]
    norm = (vecs ** 2).sum(1)
    order = np.lexsort(tuple(idx[:, ::-1].T) + (norm,))
    return np.ascontiguousarray(vecs[order[:256]], np.float32)


@dataclass
class Cb2Matrix:
    """Host container of the cb2 format (include/mlra.h mlra_cb2_create)."""
    rows: int
    cols: int
    group_size: int
    codes: np.ndarray     # uint16 [rows x cols/8]
    codebook: np.ndarray  # float32 [256 x 8]
    scales: np.ndarray    # float32 [rows x cols/group]


class Codebook2Quantizer:
    """Quantizer plugin "cb2" (quantize.hpp:91-106 interface: name(), quantize()):
    2 bits per weight as one u16 code per 8 entries (8-bit codebook index + 8
    sign bits) with a per-(row, group) scale. ``quantize`` is the offline
    nearest-codeword search on the host; ``upload`` moves the codes to HBM and
    returns an opaque DeviceQuantizedMatrix whose hook is the library's cb2
    materialize kernel."""

    def __init__(self, codebook: Optional[np.ndarray] = None):
        self.codebook = np.ascontiguousarray(
            default_cb2_codebook() if codebook is None else codebook, np.float32).reshape(256, 8)

    def name(self) -> str:
        return "cb2"

    def quantize(self, w: np.ndarray, calib=None, bits: int = 2, group_size: int = 128) -> Cb2Matrix:
        if bits != 2:
            raise MlraError(3, f"cb2: unsupported bit width {bits} (2 bits per weight)")
        w = np.asarray(w, np.float64)
        rows, cols = w.shape
        if cols % 8 or group_size % 8 or cols % group_size:
            raise MlraError(3, "cb2: cols and group size must be multiples of 8, group dividing cols")
        cb = self.codebook.astype(np.float64)
        ng = cols // group_size
        # s = group RMS: minimises the codebook's relative error on Gaussian groups
        rms = np.sqrt((w.reshape(rows, ng, group_size) ** 2).mean(-1))
        scales = np.maximum(rms, np.finfo(np.float32).tiny).astype(np.float32)
        v = w.reshape(rows, ng, group_size // 8, 8) / scales.astype(np.float64)[:, :, None, None]
        v = v.reshape(-1, 8)
        codes = np.empty(v.shape[0], np.uint16)
        cn = (cb ** 2).sum(1)
        for i in range(0, v.shape[0], 1 << 16):
            a = np.abs(v[i:i + (1 << 16)])
            d = cn[None, :] - 2.0 * a @ cb.T
            best = d.argmin(1).astype(np.uint16)
            sign = (v[i:i + (1 << 16)] < 0).astype(np.uint16)
            codes[i:i + (1 << 16)] = best | (sign << np.arange(8, 16, dtype=np.uint16)).sum(1).astype(np.uint16)
        return Cb2Matrix(rows, cols, group_size, codes.reshape(rows, cols // 8), self.codebook.copy(),
                         scales.reshape(rows, ng))

    def upload(self, m: Cb2Matrix, stream: Optional[torch.cuda.Stream] = None) -> DeviceQuantizedMatrix:
        codes = np.ascontiguousarray(m.codes, np.uint16)
        cb = np.ascontiguousarray(m.codebook, np.float32)
        sc = np.ascontiguousarray(m.scales, np.float32)
        if codes.size != m.rows * (m.cols // 8) or cb.size != 2048 or sc.size != m.rows * (m.cols // m.group_size):
            raise MlraError(7, "cb2: buffer sizes do not match the shape")
        h = C.c_void_p()
        check(lib().mlra_cb2_create(m.rows, m.cols, m.group_size, codes.ctypes.data, cb.ctypes.data,
                                    sc.ctypes.data, _stream_ptr(stream), C.byref(h)))
        return DeviceQuantizedMatrix._wrap(h, m.rows, m.cols, 2, m.group_size)


def e8p_abs_table():
    """The E8P abs-pattern table (include/mlra.h mlra_e8p_abs_table): 256 x 8 f32
    |a| patterns and the 256 odd-coordinate-sum bits."""
    a = np.empty((256, 8), np.float32)
    odd = np.empty(8, np.uint32)
    lib().mlra_e8p_abs_table(a.ctypes.data, odd.ctypes.data)
    bits = ((odd[np.arange(256) >> 5] >> (np.arange(256) & 31).astype(np.uint32)) & 1).astype(bool)
    return a, bits


def e8p_decode(codes: np.ndarray) -> np.ndarray:
    """E8P codes (u16) -> their 8-dim codewords (f64), the decode law of
    mlra_e8p_create: sign_j * |a_j| + (+1/4 if bit 15 else -1/4)."""
    a, odd = e8p_abs_table()
    c = np.asarray(codes, np.uint32).ravel()
    idx = c & 0xFF
    neg = ((c[:, None] >> (8 + np.arange(7, dtype=np.uint32))) & 1).astype(np.int64)
    n7 = (neg.sum(1) + odd[idx].astype(np.int64)) & 1
    neg = np.concatenate([neg, n7[:, None]], 1)
    sh = np.where((c >> 15) & 1, 0.25, -0.25)
    return np.where(neg == 1, -1.0, 1.0) * a[idx].astype(np.float64) + sh[:, None]


@dataclass
class E8pMatrix:
    """Host container of the e8p format (include/mlra.h mlra_e8p_create)."""
    rows: int
    cols: int
    group_size: int
    codes: np.ndarray   # uint16 [rows x cols/8]
    scales: np.ndarray  # float32 [rows x cols/group]


class E8pQuantizer:
    """Quantizer plugin "e8p" (quantize.hpp:91-106 interface): QuIP#'s E8P
    lattice codebook, 2 bits per weight — 2^16 points of E8 + 1/4 per 8
    entries, a per-(row, group) scale. ``quantize`` is the exact nearest-point
    search over the 256 abs patterns x 2 shifts (signs follow the residual,
    one flip repairs the parity constraint); ``upload`` returns an opaque
    DeviceQuantizedMatrix decoded inside the fused GEMM (whole 256-multiples)
    or through the library's e8p materialize hook."""

    def name(self) -> str:
        return "e8p"

    def quantize(self, w: np.ndarray, calib=None, bits: int = 2, group_size: int = 128) -> E8pMatrix:
        if bits != 2:
            raise MlraError(3, f"e8p: unsupported bit width {bits} (2 bits per weight)")
        w = np.asarray(w, np.float64)
        rows, cols = w.shape
        if cols % 8 or group_size % 8 or cols % group_size:
            raise MlraError(3, "e8p: cols and group size must be multiples of 8, group dividing cols")
        a, odd = e8p_abs_table()
        a = a.astype(np.float64)
        ng = cols // group_size
        # E8P codewords have RMS ~1.1 per coordinate; scale each group to match
        rms = np.sqrt((w.reshape(rows, ng, group_size) ** 2).mean(-1))
        scales = np.maximum(rms / 1.1, np.finfo(np.float32).tiny).astype(np.float32)
        v = (w.reshape(rows, ng, group_size // 8, 8) /
             scales.astype(np.float64)[:, :, None, None]).reshape(-1, 8)
        codes = np.empty(v.shape[0], np.uint16)
        for i in range(0, v.shape[0], 4096):
            y = v[i:i + 4096]
            best_err = np.full(y.shape[0], np.inf)
            best = np.zeros(y.shape[0], np.uint32)
            for shift_bit, delta in ((1, 0.25), (0, -0.25)):
                z = y - delta                              # [n, 8]
                az = np.abs(z)
                neg = z < 0                                # unconstrained signs
                err = ((az[:, None, :] - a[None, :, :]) ** 2).sum(-1)  # [n, 256]
                par = (neg.sum(1)[:, None] + odd[None, :]) & 1       # parity violated
                fix = 4.0 * (az[:, None, :] * a[None, :, :]).min(-1)  # cheapest flip
                err = err + par * fix
                k = err.argmin(1)
                e = err[np.arange(len(k)), k]
                # signs of the chosen pattern, with the parity flip applied
                jflip = (az * a[k]).argmin(1)
                s = neg.copy()
                viol = par[np.arange(len(k)), k].astype(bool)
                s[np.arange(len(k))[viol], jflip[viol]] ^= True
                code = k.astype(np.uint32) | (s[:, :7].astype(np.uint32) << np.arange(8, 15, dtype=np.uint32)).sum(1) \
                    | (np.uint32(shift_bit) << 15)
                take = e < best_err
                best_err[take] = e[take]
                best[take] = code[take]
            codes[i:i + 4096] = best.astype(np.uint16)
        return E8pMatrix(rows, cols, group_size, codes.reshape(rows, cols // 8), scales.reshape(rows, ng))

    def upload(self, m: E8pMatrix, stream: Optional[torch.cuda.Stream] = None) -> DeviceQuantizedMatrix:
        codes = np.ascontiguousarray(m.codes, np.uint16)
        sc = np.ascontiguousarray(m.scales, np.float32)
        if codes.size != m.rows * (m.cols // 8) or sc.size != m.rows * (m.cols // m.group_size):
            raise MlraError(7, "e8p: buffer sizes do not match the shape")
        h = C.c_void_p()
        check(lib().mlra_e8p_create(m.rows, m.cols, m.group_size, codes.ctypes.data, sc.ctypes.data,
                                    _stream_ptr(stream), C.byref(h)))
        return DeviceQuantizedMatrix._wrap(h, m.rows, m.cols, 2, m.group_size)


def rht(x: torch.Tensor, signs: torch.Tensor, block: int = 512, inverse: bool = False,
        out_dtype=torch.bfloat16) -> torch.Tensor:
    """Block randomized Hadamard transform (include/mlra.h mlra_rht) of a bf16
    [m x d] activation: H·diag(s)·x / sqrt(b) per b-wide block (inverse: the
    transpose, diag(s)·H·x / sqrt(b))."""
    if x.dim() != 2 or x.dtype != torch.bfloat16 or not x.is_cuda or x.stride(1) != 1:
        raise MlraError(3, "rht: expected a row-major bf16 CUDA tensor")
    if signs.dtype != torch.float32 or signs.numel() != x.shape[1] or not signs.is_contiguous():
        raise MlraError(2, "rht: signs must be a contiguous f32 vector of length cols")
    out = torch.empty(x.shape[0], x.shape[1], dtype=out_dtype, device=x.device)
    check(lib().mlra_rht(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), signs.data_ptr(),
                         int(inverse), block, out.data_ptr(), out.shape[1], _dtype_code(out_dtype),
                         _stream_ptr(None)))
    return out


def random_signs(n: int, seed: int, device="cuda") -> torch.Tensor:
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randint(0, 2, (n,), generator=g) * 2 - 1).to(torch.float32).to(device)


class IncoherentLayer:
    """QuIP#-style incoherence processing around a ModuLoRA layer (PAPER.md:224,
    :231: "orthogonal matrices multiplication in the forward and backward
    passes"). The frozen weights were quantized in the rotated basis
    W~ = U W V^T, U = H·diag(u), V = H·diag(v) (block-diagonal b-wide
    Hadamard, random signs); the adapters live in the same basis (A~ = U A,
    B~ = V B) and the bias enters as U·bias, so
        y  = U^T (layer_forward(inner, V x))           (= W x + s·(xB)A^T + bias)
        dx = V^T (layer_backward(inner, V x, ., U dy)) (dA~, dB~ from the inner layer).
    Each transform is one mlra_rht launch; the inner layer is any ModuLoraLayer
    (e8p / cb2 / affine weights)."""

    def __init__(self, inner: ModuLoraLayer, u_signs: torch.Tensor, v_signs: torch.Tensor,
                 block: int = 512):
        if inner.bias_trainable:
            raise MlraError(3, "IncoherentLayer: a trainable bias is not supported (frozen U·bias)")
        self.inner, self.u, self.v, self.block = inner, u_signs, v_signs, block

    @staticmethod
    def rotated_bias(bias: torch.Tensor, u_signs: torch.Tensor, block: int = 512) -> torch.Tensor:
        """U·bias (fp32) for the inner layer's bias."""
        return rht(bias.reshape(1, -1).to(torch.bfloat16).contiguous(), u_signs, block,
                   out_dtype=torch.float32).reshape(-1)

    def forward(self, x: torch.Tensor):
        xt = rht(x, self.v, self.block)
        yt, xb = layer_forward(self.inner, xt)
        return rht(yt, self.u, self.block, inverse=True), (xt, xb)

    def backward(self, saved, dy: torch.Tensor, da=None, db=None):
        xt, xb = saved
        dyt = rht(dy, self.u, self.block)
        dxt = layer_backward(self.inner, xt, xb, dyt, da=da, db=db)
        return rht(dxt, self.v, self.block, inverse=True)


# The QLoRA NF4 levels (Dettmers et al. 2023, "normal float 4"): the
# published f32 table, sorted, normalised to [-1, 1] with an exact 0.
NF4_LEVELS = np.array([
    -1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
    -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
    0.07958029955625534, 0.16093020141124725, 0.24611230194568634, 0.33791524171829224,
    0.44070982933044434, 0.5626170039176941, 0.7229568362236023, 1.0], np.float32)


def normal_float_levels(bits: int) -> np.ndarray:
    """2^bits "normal float" levels: NF4 for 4 bits; for 2 / 3 bits the same
    construction (quantiles of N(0, 1) at evenly spaced probabilities from
    0.9677 to 1/2 on each side, 2^(b-1) positive, 2^(b-1) - 1 negative, plus an
    exact 0), normalised by the largest magnitude."""
    if bits == 4:
        return NF4_LEVELS.copy()
    if bits not in (2, 3):
        raise MlraError(3, f"lut: unsupported bit width {bits} (2, 3 or 4)")
    from statistics import NormalDist
    inv = NormalDist().inv_cdf
    hp, hn, off = 1 << (bits - 1), (1 << (bits - 1)) - 1, 0.9677083
    pos = [inv(off + (0.5 - off) * i / hp) for i in range(hp)]
    neg = [-inv(off + (0.5 - off) * i / hn) for i in range(hn)] if hn else []
    v = np.sort(np.array(pos + neg + [0.0]))
    return (v / np.abs(v).max()).astype(np.float32)


def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """The reference's LSB-first bitstream (bitpack.cpp:68-91: code i at bit
    i*bits of a u32 word array, ceil(n*bits/32) words), vectorised on the host."""
    c = np.ascontiguousarray(codes, np.uint32).ravel()
    if c.size and int(c.max()) >> bits:
        raise MlraError(4, f"bitpack: code out of range for {bits} bits")
    nw = (c.size * bits + 31) // 32
    out = np.zeros(nw, np.uint32)
    chunk = 1 << 20  # codes per pass, a multiple of 32 (so passes start on word boundaries)
    for i in range(0, c.size, chunk):
        bitv = ((c[i:i + chunk, None] >> np.arange(bits, dtype=np.uint32)) & 1).astype(np.uint8)
        by = np.packbits(bitv.ravel(), bitorder="little")
        by = np.pad(by, (0, (-by.size) % 4))
        w = by.view("<u4")
        w0 = i * bits // 32
        out[w0:w0 + w.size] = w[:nw - w0]
    return out


@dataclass
class LutMatrix:
    """Host container of the lut format (include/mlra.h mlra_lut_create)."""
    rows: int
    cols: int
    bits: int
    group_size: int
    codes: PackedCodes    # the reference bitstream of the b-bit level indices
    levels: np.ndarray    # float32 [2^bits]
    scales: np.ndarray    # float32 [rows x cols/group], > 0


class LutQuantizer:
    """Quantizer plugin "lut" (quantize.hpp:91-106 interface: name(), quantize()):
    non-uniform levels (NF4 by default) with a per-(row, group) absmax scale,
    Ŵ = RN_f32(s · levels[c]). ``quantize`` is the offline nearest-level search
    on the host; ``upload`` returns an ordinary DeviceQuantizedMatrix whose
    materialize() and fused GEMM decode run the library's lut kernels."""

    def __init__(self, levels: Optional[np.ndarray] = None):
        self.levels = None if levels is None else np.ascontiguousarray(levels, np.float32).ravel()

    def name(self) -> str:
        return "lut"

    def levels_for(self, bits: int) -> np.ndarray:
        if self.levels is None:
            return normal_float_levels(bits)
        if self.levels.size != 1 << bits:
            raise MlraError(3, f"lut: {self.levels.size} levels for {bits} bits")
        return self.levels

    def quantize(self, w, calib=None, bits: int = 4, group_size: int = 64) -> LutMatrix:
        w = np.asarray(w, np.float64)
        if w.ndim != 2 or w.size == 0:
            raise MlraError(2, "quantize: expected a non-empty 2-D weight matrix")
        rows, cols = w.shape
        g = cols if group_size == 0 else group_size
        if g % 8 or cols % g:
            raise MlraError(3, f"lut: group size {g} must be a multiple of 8 dividing cols {cols}")
        lv = self.levels_for(bits).astype(np.float64)
        ng = cols // g
        amax = np.abs(w.reshape(rows, ng, g)).max(-1)
        scales = np.where(amax > 0, amax, 1.0).astype(np.float32)
        scales = np.maximum(scales, np.finfo(np.float32).tiny)
        x = (w.reshape(rows, ng, g) / scales.astype(np.float64)[:, :, None]).reshape(-1)
        # nearest level (levels sorted: compare against the midpoints; ties -> lower index)
        order = np.argsort(lv, kind="stable")
        srt = lv[order]
        mid = (srt[1:] + srt[:-1]) / 2
        codes = order[np.searchsorted(mid, x, side="left")].astype(np.uint32)
        return LutMatrix(rows, cols, bits, g, PackedCodes(bits, rows * cols, pack_codes(codes, bits)),
                         lv.astype(np.float32), scales.reshape(rows, ng))

    def upload(self, m: LutMatrix, stream: Optional[torch.cuda.Stream] = None) -> DeviceQuantizedMatrix:
        words = np.ascontiguousarray(m.codes.words, np.uint32)
        lv = np.ascontiguousarray(m.levels, np.float32)
        sc = np.ascontiguousarray(m.scales, np.float32)
        if lv.size != 1 << m.bits or sc.size != m.rows * (m.cols // m.group_size):
            raise MlraError(7, "lut: buffer sizes do not match the shape")
        h = C.c_void_p()
        check(lib().mlra_lut_create(m.rows, m.cols, m.bits, m.group_size, words.ctypes.data,
                                    words.size, lv.ctypes.data, sc.ctypes.data,
                                    _stream_ptr(stream), C.byref(h)))
        return DeviceQuantizedMatrix._wrap(h, m.rows, m.cols, m.bits, m.group_size)


@dataclass
class LpLinearContext:
    """lowprec_linear.hpp:85-91 (ledger replaced by ledger_bytes())."""
    q: Optional[DeviceQuantizedMatrix]
    strategy: MaterializationStrategy = MaterializationStrategy.RowMaterialize
    layer_name: str = ""
    matvec_hook: Optional[QuantizerHook] = None  # consulted under QuantizerMatvec only
    ledger: Optional["MemoryLedger"] = None      # optional (lowprec_linear.hpp:89)

    def ledger_bytes(self) -> int:
        """Bytes this strategy materializes per pass (MemoryLedger semantics)."""
        if self.q is None:
            return 0
        return int(lib().mlra_ledger_bytes(self.q.handle, int(self.strategy)))


def _hook_ptr(hook: Optional[QuantizerHook]):
    return None if hook is None else C.pointer(hook.c_hook())


def _need_q(ctx) -> DeviceQuantizedMatrix:
    if ctx.q is None:
        raise MlraError(5, "lp_linear: missing quantized weights")
    return ctx.q


def _check_act(t: torch.Tensor, cols: int, what: str) -> None:
    if t.dim() != 2 or t.stride(1) != 1:
        raise MlraError(2, f"{what}: expected a row-major 2-D tensor")
    if t.dtype != torch.bfloat16 or not t.is_cuda:
        raise MlraError(3, f"{what}: expected a bf16 CUDA tensor")
    if t.shape[1] != cols:
        raise MlraError(2, f"{what}: input cols {t.shape[1]} != {cols}")


class _Charge:
    """MaterializedBuffer (lowprec_linear.cpp:17-37): charges one pass's device
    materialization to an optional ledger for the duration of the call (the
    library frees its workspace, stream-ordered, before returning)."""

    def __init__(self, ledger, layer: str, phase: int, nbytes: int):
        self.ledger, self.layer, self.phase, self.nbytes = ledger, layer, phase, nbytes

    def __enter__(self):
        if self.ledger is not None and self.nbytes:
            self.ledger.on_alloc(self.layer, self.phase, self.nbytes)
        return self

    def __exit__(self, *exc):
        if self.ledger is not None and self.nbytes:
            self.ledger.on_free(self.layer, self.phase, self.nbytes)
        return False


def _charge(ctx: "LpLinearContext", phase: int) -> _Charge:
    led = ctx.ledger
    return _Charge(led, ctx.layer_name, phase, ctx.ledger_bytes() if led is not None else 0)


def lp_forward(ctx: LpLinearContext, x: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """lp_forward (lowprec_linear.cpp:150-196): x [m x d_in] -> [m x d_out]."""
    q = _need_q(ctx)
    _check_act(x, q.cols, "lp_forward")
    y = torch.empty(x.shape[0], q.rows, dtype=out_dtype, device=x.device)
    with _charge(ctx, 0):
        check(lib().mlra_lp_forward_ex(q.handle, int(ctx.strategy), _hook_ptr(ctx.matvec_hook),
                                       x.data_ptr(), x.stride(0), x.shape[0], y.data_ptr(),
                                       _dtype_code(out_dtype), q.rows, _stream_ptr(None)))
    return y


def lp_backward(ctx: LpLinearContext, grad_out: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """lp_backward (lowprec_linear.cpp:198-247): [m x d_out] -> [m x d_in]."""
    q = _need_q(ctx)
    _check_act(grad_out, q.rows, "lp_backward")
    dx = torch.empty(grad_out.shape[0], q.cols, dtype=out_dtype, device=grad_out.device)
    with _charge(ctx, 1):
        check(lib().mlra_lp_backward_ex(q.handle, int(ctx.strategy), _hook_ptr(ctx.matvec_hook),
                                        grad_out.data_ptr(), grad_out.stride(0), grad_out.shape[0],
                                        dx.data_ptr(), _dtype_code(out_dtype), q.cols,
                                        _stream_ptr(None)))
    return dx


kAdapterInitStd = 0.02  # lora.hpp:33


@dataclass
class LoraAdapter:
    """lora.hpp:24-31. a: [d_out x r] (zero-init), b: [d_in x r] (N(0, 0.02^2))."""
    a: torch.Tensor
    b: torch.Tensor
    rank: int
    alpha: float
    grad_a: Optional[torch.Tensor] = None
    grad_b: Optional[torch.Tensor] = None

    def scaling(self) -> float:
        return self.alpha / float(self.rank)


def mix_seed(seed: int, salt: int) -> int:
    """mix_seed (rng.hpp:52-57)."""
    return int(lib().mlra_mix_seed(seed, salt))


def gaussian(seed: int, rows: int, cols: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
    """DenseMatrix::gaussian(rows, cols, Rng(seed), mean, std) (matrix.cpp:62-67), f64 host,
    bit-identical to the reference's stream."""
    out = np.empty(rows * cols, np.float64)
    if out.size:
        lib().mlra_gaussian_fill(seed, out.ctypes.data, out.size, mean, std)
    return out.reshape(rows, cols)


def init_adapter(d_in: int, d_out: int, rank: int, alpha: float, seed: int) -> LoraAdapter:
    """init_adapter (lora.cpp:14-32): A = 0, B = gaussian(d_in x r, Rng(seed), 0, 0.02) —
    the reference's own stream (B's f64 values are bit-identical; the device copy is
    their fp32 rounding). Same errors and the same low-rank warning."""
    if rank == 0:
        raise MlraError(3, "adapter rank must be >= 1")
    if not alpha > 0.0:
        raise MlraError(3, "adapter alpha must be positive")
    if rank > min(d_in, d_out) // 2:
        import warnings
        warnings.warn(f"adapter rank {rank} exceeds half of min({d_in}, {d_out}); "
                      "the low-rank assumption is weak")
    b = gaussian(seed, d_in, rank, 0.0, kAdapterInitStd)
    return LoraAdapter(a=torch.zeros(d_out, rank, device="cuda"),
                       b=torch.from_numpy(b.astype(np.float32)).cuda(), rank=rank, alpha=alpha)


@dataclass
class ModuLoraLayer:
    """lora.hpp:40-51."""
    name: str
    weights: DeviceQuantizedMatrix
    adapter: LoraAdapter
    bias: Optional[torch.Tensor] = None  # fp32 [d_out]
    bias_trainable: bool = False
    strategy: MaterializationStrategy = MaterializationStrategy.RowMaterialize
    matvec_hook: Optional[QuantizerHook] = None  # lora.hpp:47
    grad_bias: Optional[torch.Tensor] = None
    _grads_ready: bool = field(default=False, repr=False)

    def d_in(self) -> int:
        return self.weights.cols

    def d_out(self) -> int:
        return self.weights.rows

    def _c(self) -> MlraLora:
        a = self.adapter
        if a.a.dtype != torch.float32 or a.b.dtype != torch.float32:
            raise MlraError(3, "adapter factors must be fp32")
        return MlraLora(self.weights.handle, int(self.strategy), a.rank, float(a.alpha),
                        a.a.data_ptr(), a.b.data_ptr(), _ptr(self.bias),
                        _hook_ptr(self.matvec_hook))


def make_layer(name: str, weights: DeviceQuantizedMatrix, rank: int, alpha: float, seed: int,
               strategy: MaterializationStrategy = MaterializationStrategy.RowMaterialize,
               bias_trainable: bool = False) -> ModuLoraLayer:
    """make_layer (lora.cpp:34-50)."""
    if weights is None:
        raise MlraError(5, "make_layer: null weights")
    ad = init_adapter(weights.cols, weights.rows, rank, alpha, seed)
    bias = torch.zeros(weights.rows, device="cuda")
    return ModuLoraLayer(name=name, weights=weights, adapter=ad, bias=bias,
                         bias_trainable=bias_trainable, strategy=MaterializationStrategy(strategy))


def _layer_ctx(layer: ModuLoraLayer, ledger) -> "LpLinearContext":
    return LpLinearContext(layer.weights, layer.strategy, layer.name, layer.matvec_hook, ledger)


def layer_forward(layer: ModuLoraLayer, x: torch.Tensor, out_dtype=torch.bfloat16, ledger=None):
    """layer_forward (lora.cpp:52-72). Returns (y, xb); xb = x·B is what the
    backward pass needs besides x (the tape's saved value). ``ledger``: an
    optional MemoryLedger charged with the pass's device materialization."""
    _check_act(x, layer.d_in(), f"layer '{layer.name}'")
    m = x.shape[0]
    y = torch.empty(m, layer.d_out(), dtype=out_dtype, device=x.device)
    xb = torch.empty(m, layer.adapter.rank, dtype=torch.float32, device=x.device)
    L = layer._c()
    with _charge(_layer_ctx(layer, ledger), 0):
        check(lib().mlra_lora_forward(C.byref(L), x.data_ptr(), x.stride(0), m, y.data_ptr(),
                                      _dtype_code(out_dtype), layer.d_out(), xb.data_ptr(),
                                      _stream_ptr(None)))
    return y, xb


def layer_backward(layer: ModuLoraLayer, x: torch.Tensor, xb: torch.Tensor, dy: torch.Tensor,
                   need_dx: bool = True, dx_dtype=torch.bfloat16,
                   da: Optional[torch.Tensor] = None, db: Optional[torch.Tensor] = None,
                   ledger=None):
    """Tape replay of layer_forward's records (autodiff.cpp:101-193) for the
    upstream gradient dy. Stores dA/dB (and dbias when trainable) on the layer
    (grads_of_adapter) and returns dx (None when need_dx is False). da/db may
    be caller-provided contiguous fp32 views (e.g. slices of one flat
    gradient bucket for the data-parallel all-reduce)."""
    _check_act(dy, layer.d_out(), f"layer '{layer.name}' backward")
    _check_act(x, layer.d_in(), f"layer '{layer.name}' backward")
    m = x.shape[0]
    r = layer.adapter.rank
    # the C ABI takes one token count: every per-token operand must have m rows
    # (lowprec_linear.cpp:202-206 DimensionError), on x's device
    if dy.shape[0] != m:
        raise MlraError(2, f"layer '{layer.name}' backward: grad rows {dy.shape[0]} != input rows {m}")
    if (xb.dim() != 2 or tuple(xb.shape) != (m, r) or xb.dtype != torch.float32
            or not xb.is_contiguous() or xb.device != x.device):
        raise MlraError(2, f"layer '{layer.name}' backward: xb must be a contiguous fp32 ({m}, {r}) "
                           f"tensor on {x.device}, got {tuple(xb.shape)} {xb.dtype} on {xb.device}")
    if dy.device != x.device:
        raise MlraError(2, f"layer '{layer.name}' backward: dy on {dy.device}, x on {x.device}")
    if da is None:
        da = torch.empty(layer.d_out(), r, dtype=torch.float32, device=x.device)
    if db is None:
        db = torch.empty(layer.d_in(), r, dtype=torch.float32, device=x.device)
    for t, shape in ((da, (layer.d_out(), r)), (db, (layer.d_in(), r))):
        if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
            raise MlraError(2, f"gradient buffer must be contiguous fp32 {shape}")
    dbias = torch.empty(layer.d_out(), dtype=torch.float32, device=x.device) if layer.bias_trainable else None
    dx = torch.empty(m, layer.d_in(), dtype=dx_dtype, device=x.device) if need_dx else None
    L = layer._c()
    with _charge(_layer_ctx(layer, ledger if need_dx else None), 1):
        check(lib().mlra_lora_backward(C.byref(L), x.data_ptr(), x.stride(0), xb.data_ptr(),
                                       dy.data_ptr(), dy.stride(0), m, _ptr(dx),
                                       _dtype_code(dx_dtype), layer.d_in(), da.data_ptr(),
                                       db.data_ptr(), _ptr(dbias), _stream_ptr(None)))
    layer.adapter.grad_a, layer.adapter.grad_b = da, db
    layer.grad_bias = dbias
    layer._grads_ready = True
    return dx


def grads_of_adapter(layer: ModuLoraLayer):
    """grads_of_adapter (lora.cpp:74-80): ContractError before backward."""
    if not layer._grads_ready:
        raise MlraError(5, "grads_of_adapter: called before backward()")
    return layer.adapter.grad_a, layer.adapter.grad_b


def quantized_matvec(q: DeviceQuantizedMatrix, v: torch.Tensor) -> torch.Tensor:
    """quantized_matvec (quantize.cpp:268-283): Ŵ·v for one vector (as bf16
    operands into the fused kernel, fp32 result)."""
    v = v.reshape(1, -1).to(torch.bfloat16).contiguous()
    return lp_forward(LpLinearContext(q, MaterializationStrategy.QuantizerMatvec), v, torch.float32)[0]


def quantized_matvec_transposed(q: DeviceQuantizedMatrix, v: torch.Tensor) -> torch.Tensor:
    """quantized_matvec_transposed (quantize.cpp:285-300): Ŵᵀ·v."""
    v = v.reshape(1, -1).to(torch.bfloat16).contiguous()
    return lp_backward(LpLinearContext(q, MaterializationStrategy.QuantizerMatvec), v, torch.float32)[0]


def unpack_codes(words: np.ndarray, count: int, bits: int) -> np.ndarray:
    """unpack (bitpack.cpp:93-104): the reference bitstream back to u32 codes,
    vectorised on the host (code i at bit i*bits, LSB first)."""
    w = np.ascontiguousarray(words, np.uint32)
    if w.size != (count * bits + 31) // 32:
        raise MlraError(7, f"bitpack: corrupted length metadata: {w.size} words for {count} codes")
    if count == 0:
        return np.zeros(0, np.uint32)
    bitv = np.unpackbits(w.view(np.uint8), bitorder="little")[:count * bits]
    return (bitv.reshape(count, bits).astype(np.uint32) << np.arange(bits, dtype=np.uint32)).sum(
        1, dtype=np.uint32)


class LpLinearFunction(torch.autograd.Function):
    """LpLinearFunction (lowprec_linear.hpp:96-112): the frozen quantized linear
    alone on the tape — forward y = x·Ŵᵀ, backward dX = dY·Ŵ (re-dequantized in
    the fused kernel, never cached); no gradient for the quantized weights."""

    @staticmethod
    def forward(ctx, x, lp_ctx: "LpLinearContext"):
        ctx.lp = lp_ctx
        return lp_forward(lp_ctx, x.to(torch.bfloat16).contiguous(), torch.float32)

    @staticmethod
    def backward(ctx, dy):
        dx = lp_backward(ctx.lp, dy.to(torch.bfloat16).contiguous(), torch.float32)
        return dx, None


class ModuLoraLinearFunction(torch.autograd.Function):
    """The reference's CustomFunction plug-in point (autodiff.hpp:77-89) as a
    torch.autograd.Function: forward saves only x and xb (never Ŵ); backward
    re-dequantizes inside the fused kernel."""

    @staticmethod
    def forward(ctx, x, a, b, bias, layer: ModuLoraLayer):
        y, xb = layer_forward(layer, x)
        ctx.layer = layer
        ctx.save_for_backward(x, xb)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, xb = ctx.saved_tensors
        layer = ctx.layer
        dx = layer_backward(layer, x, xb, dy.contiguous(), need_dx=ctx.needs_input_grad[0])
        da, db = layer.adapter.grad_a, layer.adapter.grad_b
        return dx, da, db, layer.grad_bias, None
