"""The C-ABI data-parallel exchange (mlra_dp_* / mlra_allreduce_lora_grads,
NCCL loaded by libmlra). Only one GPU is available to the tests, so the
communicator is world size 1 (a sum over one rank is the identity) — the
multi-rank reduction semantics are covered by tests/test_dp_gloo.py."""
import pytest
import torch

from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200.dp import GradBucket, NcclGradExchange

pytestmark = pytest.mark.gpu


def test_nccl_exchange_world_one():
    bucket = GradBucket.create([("l.dA", (300, 16)), ("l.dB", (200, 16))], "cuda")
    bucket.flat.copy_(torch.randn(bucket.flat.numel()))
    before = bucket.flat.clone()
    ex = NcclGradExchange(0, 1, NcclGradExchange.unique_id())
    ex.allreduce(bucket)
    torch.cuda.synchronize()
    assert torch.equal(bucket.flat, before)


def test_nccl_exchange_bad_rank():
    with pytest.raises(MlraError) as e:
        NcclGradExchange(2, 1, NcclGradExchange.unique_id())
    assert e.value.kind == "ConfigError"
