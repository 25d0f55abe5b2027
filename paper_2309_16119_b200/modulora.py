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
    QuantizedMatrix::validate, quantize.cpp:82-115)."""

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


def dequantize_row(q: DeviceQuantizedMatrix, row: int, dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """dequantize_row (quantize.cpp:139-161); RangeError past the last row."""
    out = torch.empty(1, q.cols, dtype=dtype, device="cuda")
    check(lib().mlra_materialize_rows(q.handle, row, 1, out.data_ptr(), _dtype_code(dtype),
                                      q.cols, _stream_ptr(None)))
    return out[0]


@dataclass
class LpLinearContext:
    """lowprec_linear.hpp:85-91 (ledger replaced by ledger_bytes())."""
    q: Optional[DeviceQuantizedMatrix]
    strategy: MaterializationStrategy = MaterializationStrategy.RowMaterialize
    layer_name: str = ""

    def ledger_bytes(self) -> int:
        """Bytes this strategy materializes per pass (MemoryLedger semantics)."""
        if self.q is None:
            return 0
        return int(lib().mlra_ledger_bytes(self.q.handle, int(self.strategy)))


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


def lp_forward(ctx: LpLinearContext, x: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """lp_forward (lowprec_linear.cpp:150-196): x [m x d_in] -> [m x d_out]."""
    q = _need_q(ctx)
    _check_act(x, q.cols, "lp_forward")
    y = torch.empty(x.shape[0], q.rows, dtype=out_dtype, device=x.device)
    check(lib().mlra_lp_forward(q.handle, int(ctx.strategy), x.data_ptr(), x.stride(0),
                                x.shape[0], y.data_ptr(), _dtype_code(out_dtype), q.rows,
                                _stream_ptr(None)))
    return y


def lp_backward(ctx: LpLinearContext, grad_out: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """lp_backward (lowprec_linear.cpp:198-247): [m x d_out] -> [m x d_in]."""
    q = _need_q(ctx)
    _check_act(grad_out, q.rows, "lp_backward")
    dx = torch.empty(grad_out.shape[0], q.cols, dtype=out_dtype, device=grad_out.device)
    check(lib().mlra_lp_backward(q.handle, int(ctx.strategy), grad_out.data_ptr(),
                                 grad_out.stride(0), grad_out.shape[0], dx.data_ptr(),
                                 _dtype_code(out_dtype), q.cols, _stream_ptr(None)))
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


def init_adapter(d_in: int, d_out: int, rank: int, alpha: float, seed: int) -> LoraAdapter:
    """init_adapter (lora.cpp:14-32): same shapes, init law and errors. The
    Gaussian stream comes from torch (not the reference mt19937_64 stream)."""
    if rank == 0:
        raise MlraError(3, "adapter rank must be >= 1")
    if not alpha > 0.0:
        raise MlraError(3, "adapter alpha must be positive")
    g = torch.Generator(device="cpu").manual_seed(seed)
    b = (torch.randn(d_in, rank, generator=g, dtype=torch.float64) * kAdapterInitStd).float()
    return LoraAdapter(a=torch.zeros(d_out, rank, device="cuda"), b=b.cuda(), rank=rank,
                       alpha=alpha)


@dataclass
class ModuLoraLayer:
    """lora.hpp:40-51."""
    name: str
    weights: DeviceQuantizedMatrix
    adapter: LoraAdapter
    bias: Optional[torch.Tensor] = None  # fp32 [d_out]
    bias_trainable: bool = False
    strategy: MaterializationStrategy = MaterializationStrategy.RowMaterialize
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
                        a.a.data_ptr(), a.b.data_ptr(), _ptr(self.bias))


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


def layer_forward(layer: ModuLoraLayer, x: torch.Tensor, out_dtype=torch.bfloat16):
    """layer_forward (lora.cpp:52-72). Returns (y, xb); xb = x·B is what the
    backward pass needs besides x (the tape's saved value)."""
    _check_act(x, layer.d_in(), f"layer '{layer.name}'")
    m = x.shape[0]
    y = torch.empty(m, layer.d_out(), dtype=out_dtype, device=x.device)
    xb = torch.empty(m, layer.adapter.rank, dtype=torch.float32, device=x.device)
    L = layer._c()
    check(lib().mlra_lora_forward(C.byref(L), x.data_ptr(), x.stride(0), m, y.data_ptr(),
                                  _dtype_code(out_dtype), layer.d_out(), xb.data_ptr(),
                                  _stream_ptr(None)))
    return y, xb


def layer_backward(layer: ModuLoraLayer, x: torch.Tensor, xb: torch.Tensor, dy: torch.Tensor,
                   need_dx: bool = True, dx_dtype=torch.bfloat16,
                   da: Optional[torch.Tensor] = None, db: Optional[torch.Tensor] = None):
    """Tape replay of layer_forward's records (autodiff.cpp:101-193) for the
    upstream gradient dy. Stores dA/dB (and dbias when trainable) on the layer
    (grads_of_adapter) and returns dx (None when need_dx is False). da/db may
    be caller-provided contiguous fp32 views (e.g. slices of one flat
    gradient bucket for the data-parallel all-reduce)."""
    _check_act(dy, layer.d_out(), f"layer '{layer.name}' backward")
    _check_act(x, layer.d_in(), f"layer '{layer.name}' backward")
    m = x.shape[0]
    r = layer.adapter.rank
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
