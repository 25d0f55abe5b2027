"""Data parallelism over token micro-batches.

The frozen packed weights, grids and bias are replicated; tokens are sharded
across ranks; the only exchange per step is a sum all-reduce of the LoRA
gradients {dA [d_out x r], dB [d_in x r]} (+ dbias when trainable) — dA and dB
are sums over tokens (autodiff.cpp:153-155), so the sum of per-shard gradients
equals the full-batch gradient. The reference has no distribution at all
(SPEC.md:453); this is the B200 build's own plumbing over torch.distributed
(NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import torch


def shard_tokens(m: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous token range [begin, end) of `rank` (sizes differ by <= 1)."""
    base, extra = divmod(m, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


@dataclass
class GradBucket:
    """One flat fp32 buffer holding every LoRA gradient of a step, so the
    data-parallel exchange is a single all-reduce (one NCCL launch, latency
    bound at these sizes: 2-16 MB per step)."""

    flat: torch.Tensor
    views: Dict[str, torch.Tensor]

    @staticmethod
    def create(shapes: Sequence[Tuple[str, Tuple[int, ...]]], device) -> "GradBucket":
        total = sum(int(torch.tensor(s).prod()) for _, s in shapes)
        flat = torch.zeros(total, dtype=torch.float32, device=device)
        views, o = {}, 0
        for name, s in shapes:
            n = int(torch.tensor(s).prod())
            views[name] = flat[o:o + n].view(*s)
            o += n
        return GradBucket(flat, views)

    @staticmethod
    def for_layers(layers: List, device) -> "GradBucket":
        """dA/dB (and dbias if trainable) of each ModuLoRA layer, in order."""
        shapes = []
        for L in layers:
            r = L.adapter.rank
            shapes.append((f"{L.name}.dA", (L.d_out(), r)))
            shapes.append((f"{L.name}.dB", (L.d_in(), r)))
            if L.bias_trainable:
                shapes.append((f"{L.name}.dbias", (L.d_out(),)))
        return GradBucket.create(shapes, device)

    def slice_of(self, names: Sequence[str]) -> torch.Tensor:
        """The contiguous span of the flat buffer covering the named views."""
        base = self.flat.data_ptr()
        es = self.flat.element_size()
        lo = min((self.views[n].data_ptr() - base) // es for n in names)
        hi = max((self.views[n].data_ptr() - base) // es + self.views[n].numel() for n in names)
        return self.flat[lo:hi]

    def allreduce_async(self, names: Sequence[str], group=None):
        """Start the sum all-reduce of one layer's gradients (their span of the
        bucket) as soon as they exist, so it overlaps the remaining backward;
        returns the work handle (None when not distributed)."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            return dist.all_reduce(self.slice_of(names), op=dist.ReduceOp.SUM, group=group,
                                   async_op=True)
        return None

    def allreduce(self, group=None) -> None:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


class NcclGradExchange:
    """The same exchange through libmlra's own C ABI (mlra_dp_* /
    mlra_allreduce_lora_grads: NCCL loaded by the library) for processes that
    do not run torch.distributed — the path a C++ caller of include/mlra.h
    uses. Rank 0 makes the id (``unique_id()``) and shares it out of band."""

    def __init__(self, rank: int, world: int, uid: bytes):
        import ctypes as C
        from ._lib import check, lib
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self._buf = C.create_string_buffer(uid, 128)
        h = C.c_void_p()
        check(lib().mlra_dp_init(rank, world, self._buf, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from ._lib import check, lib
        b = C.create_string_buffer(128)
        check(lib().mlra_dp_unique_id(b))
        return b.raw

    def allreduce(self, bucket: GradBucket, stream=None) -> None:
        from ._lib import check, lib
        s = stream if stream is not None else torch.cuda.current_stream()
        check(lib().mlra_allreduce_lora_grads(self._h, bucket.flat.data_ptr(), bucket.flat.numel(),
                                              s.cuda_stream))

    def __del__(self):
        try:
            from . import _lib
            if getattr(self, "_h", None) is not None and self._h.value and _lib._lib is not None:
                _lib.lib().mlra_dp_destroy(self._h)
                self._h = None
        except Exception:
            pass
