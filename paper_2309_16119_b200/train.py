"""The step either side of the layer: adapter optimizer on the device and the
data-parallel training step over a stack of ModuLoRA linears.

  reference (train.hpp / train.cpp)          here
  ---------------------------------------    --------------------------------------------------
  TrainConfig (+validate), LrSchedule,       TrainConfig, LrSchedule, parse_schedule, lr_at
  parse_schedule, lr_at (:14-63)             (host scalars; same formulas, same libm)
  AdamW(beta1, beta2, eps, wd), step()       AdamW: f64 masters + moments in HBM, one fused
  (:75-134)                                  kernel per step over the flat bucket
                                             (mlra_adamw_step), bit-identical f64 arithmetic
  trainable_param_names order                AdapterParams: {name.A, name.B[, name.bias]} per
  (model.cpp:186-197)                        layer, views into one flat fp32 buffer
  train() loop (:136-...)                    LinearStackTrainer.step: fwd of every layer, bwd in
                                             reverse with each layer's gradients all-reduced as
                                             soon as they exist (overlapping the next layer's
                                             backward), then one AdamW launch
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import _lib
from ._lib import MlraError, check, lib
from .dp import GradBucket
from .modulora import ModuLoraLayer, _stream_ptr, layer_backward, layer_forward


class LrSchedule(enum.IntEnum):
    """train.hpp:20."""
    Constant = 0
    Cosine = 1
    Linear = 2


def parse_schedule(name: str) -> LrSchedule:
    """train.cpp:14-20."""
    try:
        return {"constant": LrSchedule.Constant, "cosine": LrSchedule.Cosine,
                "linear": LrSchedule.Linear}[name]
    except KeyError:
        raise MlraError(3, f"unknown schedule '{name}' (expected constant, cosine or linear)") from None


@dataclass
class TrainConfig:
    """train.hpp:25-38 (validate: train.cpp:31-44)."""
    steps: int = 100
    batch_size: int = 32
    lr: float = 1e-2
    weight_decay: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 1
    warmup_ratio: float = 0.0
    schedule: LrSchedule = LrSchedule.Constant

    def validate(self) -> None:
        if self.lr <= 0.0:
            raise MlraError(3, "train config: lr must be > 0")
        if not (0.0 <= self.warmup_ratio < 1.0):
            raise MlraError(3, "train config: warmup_ratio must be in [0, 1)")
        if self.batch_size == 0:
            raise MlraError(3, "train config: batch_size must be >= 1")
        if self.weight_decay < 0.0:
            raise MlraError(3, "train config: weight_decay must be >= 0")
        if not (0.0 <= self.beta1 < 1.0) or not (0.0 <= self.beta2 < 1.0):
            raise MlraError(3, "train config: betas must be in [0, 1)")
        if self.eps <= 0.0:
            raise MlraError(3, "train config: eps must be > 0")


def lr_at(config: TrainConfig, step: int) -> float:
    """train.cpp:46-63 (Python floats are IEEE f64; math.cos is the same libm cos)."""
    warmup = int(config.warmup_ratio * float(config.steps))
    if warmup > 0 and step < warmup:
        return config.lr * float(step + 1) / float(warmup)
    if config.schedule == LrSchedule.Constant:
        return config.lr
    span = max(1.0, float(config.steps - warmup))
    p = float(step - warmup) / span
    if config.schedule == LrSchedule.Cosine:
        return config.lr * 0.5 * (1.0 + math.cos(3.14159265358979323846 * p))
    return config.lr * (1.0 - p)


class AdamW:
    """AdamW with decoupled weight decay (train.hpp:51-70, train.cpp:75-134).

    Holds, per flat parameter bucket, f64 master values and f64 moments in HBM
    ("allocated on first use", train.cpp:86-93). ``step`` runs one fused
    device kernel (mlra_adamw_step) that applies the reference's f64 update
    bit-for-bit to every parameter and writes the fp32 working copy back into
    the parameters the layer kernels read."""

    def __init__(self, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0):
        self.cfg = _lib.MlraAdamw(beta1, beta2, eps, weight_decay)
        self.master: Optional[torch.Tensor] = None
        self.m: Optional[torch.Tensor] = None
        self.v: Optional[torch.Tensor] = None
        self._sizes: Optional[List[int]] = None

    @classmethod
    def from_config(cls, c: TrainConfig) -> "AdamW":
        return cls(c.beta1, c.beta2, c.eps, c.weight_decay)

    def step(self, flat_params: torch.Tensor, sizes: Sequence[int], names: Sequence[str],
             flat_grads: torch.Tensor, step_index: int, lr: float, check_finite: bool = True):
        """One update over the parameters laid out back to back in ``flat_params``
        (fp32 working copy, or f64) with gradients ``flat_grads`` (fp32 or f64,
        same layout). Raises NumericError naming the first parameter with a
        non-finite gradient (earlier ones are updated, it and later ones not),
        as train.cpp:113-117; ``check_finite=False`` keeps the call asynchronous
        and returns the device int holding that index instead."""
        sizes = [int(s) for s in sizes]
        if len(sizes) != len(names):
            raise MlraError(5, "adamw: params/names size mismatch")
        if self._sizes is None:
            self._sizes = sizes
            n = sum(sizes)
            dev = flat_params.device
            self.master = flat_params.detach().to(torch.float64).clone()
            self.m = torch.zeros(n, dtype=torch.float64, device=dev)
            self.v = torch.zeros(n, dtype=torch.float64, device=dev)
        elif sizes != self._sizes:
            raise MlraError(5, "adamw: parameter list changed between steps")
        n = sum(sizes)
        if flat_params.numel() != n or flat_grads.numel() != n:
            raise MlraError(2, "adamw: bucket sizes do not match the parameter list")
        offs = (C.c_int64 * (len(sizes) + 1))()
        o = 0
        for i, s in enumerate(sizes):
            offs[i] = o
            o += s
        offs[len(sizes)] = o
        gdt = {torch.float32: _lib.F32, torch.float64: _lib.F64}.get(flat_grads.dtype)
        if gdt is None or not flat_grads.is_contiguous():
            raise MlraError(3, "adamw: gradients must be a contiguous f32 or f64 bucket")
        p32 = flat_params if flat_params.dtype == torch.float32 else None
        bad = None if check_finite else torch.empty(1, dtype=torch.int32, device=flat_params.device)
        try:
            check(lib().mlra_adamw_step(
                C.byref(self.cfg), step_index, lr, len(sizes), offs, self.master.data_ptr(),
                self.m.data_ptr(), self.v.data_ptr(), flat_grads.data_ptr(), gdt,
                None if p32 is None else p32.data_ptr(), None if bad is None else bad.data_ptr(),
                _stream_ptr(None)))
        except MlraError as e:
            if e.kind == "NumericError":  # name the parameter, as train.cpp:113-117 does
                i = int(str(e).split("#")[1].split()[0])
                e.args = (f"NumericError: adamw: non-finite gradient for parameter "
                          f"'{names[i]}' at step {step_index}",)
                e.param_index = i
            raise
        finally:
            if flat_params.dtype == torch.float64:
                flat_params.copy_(self.master)
        return bad


class AdapterParams:
    """The trainable parameters of a list of layers in the reference's order
    (model.cpp:186-197: name.A, name.B[, name.bias] per layer) as views into one
    flat fp32 buffer, so the optimizer is one launch and the gradient bucket
    (dp.GradBucket.for_layers, same order) lines up element for element."""

    def __init__(self, layers: Sequence[ModuLoraLayer]):
        self.layers = list(layers)
        self.names: List[str] = []
        self.sizes: List[int] = []
        srcs = []
        for L in self.layers:
            for nm, t in ((".A", L.adapter.a), (".B", L.adapter.b)) + (
                    ((".bias", L.bias),) if L.bias_trainable else ()):
                self.names.append(L.name + nm)
                self.sizes.append(t.numel())
                srcs.append(t)
        dev = srcs[0].device
        self.flat = torch.empty(sum(self.sizes), dtype=torch.float32, device=dev)
        o = 0
        for L in self.layers:
            r = L.adapter.rank
            for attr, shape in (("a", (L.d_out(), r)), ("b", (L.d_in(), r))):
                n = shape[0] * shape[1]
                view = self.flat[o:o + n].view(*shape)
                view.copy_(getattr(L.adapter, attr))
                setattr(L.adapter, attr, view)
                o += n
            if L.bias_trainable:
                view = self.flat[o:o + L.d_out()]
                view.copy_(L.bias)
                L.bias = view
                o += L.d_out()


class LinearStackTrainer:
    """A data-parallel training step over a stack of ModuLoRA linears (the
    LLaMA decoder-layer linears of BASELINE configs[2]: Q, K, V, O, gate, up,
    down): forward through every layer, backward in reverse record order
    (autodiff.cpp:101-139) with upstream gradients supplied per layer, each
    layer's LoRA gradients all-reduced (async, NCCL) the moment its backward
    finishes so the exchange overlaps the remaining backward work, then one
    AdamW launch over the whole adapter bucket.

    The non-linear glue between the linears (attention, norms, activations)
    is not on the hot path — callers pass each layer's input and
    upstream gradient."""

    def __init__(self, layers: Sequence[ModuLoraLayer], config: TrainConfig, group=None):
        config.validate()
        self.layers = list(layers)
        self.config = config
        self.params = AdapterParams(self.layers)
        dev = self.params.flat.device
        self.grads = GradBucket.for_layers(self.layers, dev)
        self.opt = AdamW.from_config(config)
        self.group = group
        self.step_index = 0

    def _world(self) -> int:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def forward(self, xs: Sequence[torch.Tensor]):
        return [layer_forward(L, x) for L, x in zip(self.layers, xs)]

    def backward(self, xs, xbs, dys, need_dx: bool = False):
        """Reverse order; returns the dX list (None entries when not needed)."""
        world = self._world()
        works, dxs = [], [None] * len(self.layers)
        for i in reversed(range(len(self.layers))):
            L = self.layers[i]
            dxs[i] = layer_backward(L, xs[i], xbs[i], dys[i], need_dx=need_dx,
                                    da=self.grads.views[f"{L.name}.dA"],
                                    db=self.grads.views[f"{L.name}.dB"])
            if L.bias_trainable and L.grad_bias is not None:
                self.grads.views[f"{L.name}.dbias"].copy_(L.grad_bias)
            if world > 1:
                names = [f"{L.name}.dA", f"{L.name}.dB"] + (
                    [f"{L.name}.dbias"] if L.bias_trainable else [])
                works.append(self.grads.allreduce_async(names, group=self.group))
        for w in works:
            if w is not None:
                w.wait()
        return dxs

    def optimizer_step(self, check_finite: bool = True):
        lr = lr_at(self.config, self.step_index)
        bad = self.opt.step(self.params.flat, self.params.sizes, self.params.names,
                            self.grads.flat, self.step_index, lr, check_finite=check_finite)
        self.step_index += 1
        return bad

    def step(self, xs, dys, need_dx: bool = False, check_finite: bool = True):
        outs = self.forward(xs)
        xbs = [xb for _, xb in outs]
        dxs = self.backward(xs, xbs, dys, need_dx=need_dx)
        self.optimizer_step(check_finite=check_finite)
        return [y for y, _ in outs], dxs
