"""The decoder-layer caller of the hot path: the reference's
parity transformer (model.cpp:226-257, `transformer_forward`) and its loss
(model.cpp:259-292, `model_loss`) on the device, batched over sequences, with a
data-parallel training step (fwd, bwd, per-layer async all-reduce, AdamW).

The seven ModuLoRA linears (attn_q, attn_k, attn_v, attn_o, mlp_in, mlp_out,
head; model.cpp:21-23) run through libmlra (fused dequant + tcgen05 GEMM, the
skinny LoRA kernels). The glue between them — layer_norm without affine
parameters (autodiff.cpp:272-313), softmax attention over the whole sequence,
erf-GELU (autodiff.cpp:232-241), mean pooling (the 1/seq pool row,
model.cpp:251-255) and cross entropy (autodiff.cpp:367-410) — is torch
autograd in fp32: plumbing off the hot path, as the reference's tape ops are.

The reference runs one sequence per tape pass and averages the per-sample
losses; here the B sequences of a batch are one pass (m = B·seq tokens per
linear, batched attention), which is the same function of the same inputs.
Parity against the reference's own forward + backward on a reference-made
checkpoint: tests/test_model.py.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import torch
import torch.nn.functional as F

from ._lib import MlraError
from .dp import GradBucket
from .modulora import ModuLoraLayer, layer_backward, layer_forward
from .train import AdamW, AdapterParams, TrainConfig, lr_at

LAYER_NAMES = ("attn_q", "attn_k", "attn_v", "attn_o", "mlp_in", "mlp_out", "head")


class _Linear(torch.autograd.Function):
    """One ModuLoRA linear on the tape: forward saves x and xb only (Ŵ is
    re-dequantized inside the backward GEMM, lowprec_linear.cpp:198-247); the
    backward writes dA / dB straight into the trainer's gradient bucket and
    starts that layer's all-reduce while the rest of the backward runs."""

    @staticmethod
    def forward(ctx, x, anchor, layer: ModuLoraLayer, sink):
        # x is the fp32 activation: the bf16 operand is made here, so the
        # fp32 dx returned by backward matches the input's dtype and reaches
        # the residual stream unrounded
        x16 = x.to(torch.bfloat16).contiguous()
        y, xb = layer_forward(layer, x16, out_dtype=torch.float32)
        ctx.layer, ctx.sink = layer, sink
        ctx.save_for_backward(x16, xb)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, xb = ctx.saved_tensors
        L, sink = ctx.layer, ctx.sink
        da = db = None
        if sink is not None:
            da, db = sink.views[f"{L.name}.dA"], sink.views[f"{L.name}.dB"]
        dx = layer_backward(L, x, xb, dy.to(torch.bfloat16).contiguous(),
                            need_dx=ctx.needs_input_grad[0], dx_dtype=torch.float32, da=da, db=db)
        if sink is not None:
            if L.bias_trainable and L.grad_bias is not None:
                sink.views[f"{L.name}.dbias"].copy_(L.grad_bias)
            sink.layer_done(L)
        return dx, None, None, None


class ParityTransformer:
    """ToyModel of kind parity_transformer (model.hpp:14-66) over device
    layers, e.g. ``Checkpoint.to_layers()`` of a reference-made .mlra."""

    def __init__(self, layers: Sequence[ModuLoraLayer], ln_eps: float = 1e-5):
        layers = list(layers)
        if len(layers) != len(LAYER_NAMES):
            raise MlraError(5, f"transformer_forward: expected {len(LAYER_NAMES)} layers")
        for L, nm in zip(layers, LAYER_NAMES):
            if L.name != nm:
                raise MlraError(3, f"parity_transformer: layer must be '{nm}', got '{L.name}'")
        if not ln_eps > 0.0:
            raise MlraError(3, "layer_norm: eps must be positive")
        self.layers = layers
        self.ln_eps = float(ln_eps)
        self.d_model = layers[0].d_in()
        self.sink = None  # set by TransformerTrainer
        # the adapters live outside torch autograd (their gradients come from the
        # kernels); this leaf makes every linear's output part of the tape
        self._anchor = torch.zeros((), device=layers[0].adapter.a.device, requires_grad=True)

    def _lin(self, i: int, h: torch.Tensor) -> torch.Tensor:
        lead = h.shape[:-1]
        x = h.reshape(-1, h.shape[-1]).float()
        y = _Linear.apply(x, self._anchor, self.layers[i], self.sink)
        return y.reshape(*lead, y.shape[-1])

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: [B, seq, d_model] fp32 -> logits [B, n_classes] (model.cpp:226-257)."""
        if x.dim() == 2:
            x = x.unsqueeze(0)
        if x.dim() != 3 or x.shape[-1] != self.d_model:
            raise MlraError(2, f"transformer_forward: input must be [B, seq, {self.d_model}]")
        x = x.float()
        d = self.d_model
        inv_sqrt_d = 1.0 / math.sqrt(float(self.layers[0].d_out()))
        ln1 = F.layer_norm(x, (d,), eps=self.ln_eps)
        q, k, v = self._lin(0, ln1), self._lin(1, ln1), self._lin(2, ln1)
        scores = torch.matmul(q, k.transpose(1, 2)) * inv_sqrt_d
        ctx = torch.matmul(torch.softmax(scores, dim=-1), v)
        h = x + self._lin(3, ctx)
        ln2 = F.layer_norm(h, (h.shape[-1],), eps=self.ln_eps)
        inner = F.gelu(self._lin(4, ln2))  # erf form, as autodiff.cpp:232-241
        h2 = h + self._lin(5, inner)
        pooled = h2.mean(dim=1)  # the 1/seq pool row
        return self._lin(6, pooled)

    def loss(self, x: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """model_loss for parity (model.cpp:275-292): mean cross entropy."""
        logits = self.forward(x)
        labels = labels.to(device=logits.device, dtype=torch.long).reshape(-1)
        if labels.numel() != logits.shape[0]:
            raise MlraError(2, f"cross_entropy: {labels.numel()} labels for {logits.shape[0]} rows")
        if labels.numel() and (int(labels.min()) < 0 or int(labels.max()) >= logits.shape[1]):
            raise MlraError(4, "cross_entropy: label out of range")
        return F.cross_entropy(logits, labels)


class _Sink:
    """The trainer's gradient bucket as seen from the tape: per-layer views and
    the async all-reduce started when a layer's backward finishes."""

    def __init__(self, bucket: GradBucket, group):
        self.bucket = bucket
        self.views = bucket.views
        self.group = group
        self.works = []
        self.weight = None  # (local batch, global-batch tensor, its all-reduce) when distributed

    def layer_done(self, L: ModuLoraLayer) -> None:
        names = [f"{L.name}.dA", f"{L.name}.dB"] + ([f"{L.name}.dbias"] if L.bias_trainable else [])
        if self.weight is not None:
            n_local, total, cw = self.weight
            if cw is not None:
                cw.wait()
                self.weight = (n_local, total, None)
            self.bucket.slice_of(names).mul_(n_local / total)  # device-side, no host sync
        w = self.bucket.allreduce_async(names, group=self.group)
        if w is not None:
            self.works.append(w)

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        self.works = []


class TransformerTrainer:
    """One data-parallel training step of the parity transformer (train.cpp:136-176
    per step: zero grads, loss, backward, AdamW): each rank runs its share of the
    batch; gradients are sum-all-reduced per layer during the backward, each
    rank's contribution weighted by local_batch / global_batch, i.e. the
    gradient of the global mean loss even when the local batches differ."""

    def __init__(self, model: ParityTransformer, config: TrainConfig, group=None):
        config.validate()
        self.model = model
        self.config = config
        self.params = AdapterParams(model.layers)
        self.grads = GradBucket.for_layers(model.layers, self.params.flat.device)
        self.opt = AdamW.from_config(config)
        self.group = group
        self.sink = _Sink(self.grads, group)
        self.step_index = 0

    def _world(self) -> int:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def loss_and_grads(self, x: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """Forward + backward; leaves the (world-averaged) gradients in
        ``self.grads.flat`` and returns the local loss (a device scalar)."""
        world = self._world()
        count = None
        if world > 1:
            import torch.distributed as dist
            n_local = x.shape[0] if x.dim() == 3 else 1
            count = torch.tensor([float(n_local)], device=self.grads.flat.device)
            cw = dist.all_reduce(count, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            # the local mean loss's gradient, weighted by this rank's share of the
            # global batch: the per-layer sums then form the global mean's gradient
            self.sink.weight = (n_local, count, cw)
        self.model.sink = self.sink
        try:
            loss = self.model.loss(x, labels)
            loss.backward()
        finally:
            self.model.sink = None
        self.sink.wait()
        self.sink.weight = None
        return loss.detach()

    def step(self, x: torch.Tensor, labels: torch.Tensor, check_finite: bool = True) -> torch.Tensor:
        loss = self.loss_and_grads(x, labels)
        lr = lr_at(self.config, self.step_index)
        self.opt.step(self.params.flat, self.params.sizes, self.params.names, self.grads.flat,
                      self.step_index, lr, check_finite=check_finite)
        self.step_index += 1
        return loss

    def param_grads(self) -> List[torch.Tensor]:
        """dA, dB (, dbias) per layer in trainable_params order (model.cpp:186-197)."""
        return [self.grads.views[n.replace(".A", ".dA").replace(".B", ".dB").replace(".bias", ".dbias")]
                for n in self.params.names]
