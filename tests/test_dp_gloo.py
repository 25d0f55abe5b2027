"""Data-parallel exchange on CPU (gloo, world_size 2): token-sharded per-rank
LoRA gradients, summed by the GradBucket all-reduce, equal the full-batch
gradients of the reference algebra (oracle), and the token sharding covers
every token exactly once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_16119_b200.dp import GradBucket, shard_tokens


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from oracle import oracle as orc
    d_out, d_in, r, m, alpha = 24, 40, 4, 11, 8.0
    words, sc, z = orc.quantize_rtn(orc.gaussian(1, d_out, d_in, 0, 0.02), 3, 8)
    w = orc.dequantize(words, d_out, d_in, 3, 8, sc, z)
    a = orc.gaussian(2, d_out, r, 0, 0.5)
    b = orc.gaussian(3, d_in, r, 0, 0.02)
    x = orc.gaussian(4, m, d_in)
    g = orc.gaussian(5, m, d_out)
    return w, a, b, alpha, x, g


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, a, b, alpha, x, g = _case()
    lo, hi = shard_tokens(x.shape[0], rank, world)
    _, xb = orc.layer_forward(w, a, b, alpha, None, x[lo:hi])
    _, da, db, dbias = orc.layer_backward(w, a, b, alpha, x[lo:hi], xb, g[lo:hi],
                                          need_dx=False, need_dbias=True)
    bucket = GradBucket.create([("l.dA", da.shape), ("l.dB", db.shape), ("l.dbias", dbias.shape)],
                               "cpu")
    bucket.views["l.dA"].copy_(torch.from_numpy(da))
    bucket.views["l.dB"].copy_(torch.from_numpy(db))
    bucket.views["l.dbias"].copy_(torch.from_numpy(dbias))
    if os.environ.get("MLRA_TEST_ASYNC"):
        # per-layer form used by bench.py / LinearStackTrainer: slices all-reduced
        # asynchronously as they become ready, then waited on
        works = [bucket.allreduce_async(["l.dbias"]), bucket.allreduce_async(["l.dA", "l.dB"])]
        for wk in works:
            wk.wait()
    else:
        bucket.allreduce()
    if rank == 0:
        out.put({k: v.numpy().copy() for k, v in bucket.views.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_shard_tokens_partition():
    for m in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            ranges = [shard_tokens(m, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            sizes = [e - s for s, e in ranges]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("mode", ["flat", "async_slices"])
def test_gloo_allreduce_matches_full_batch(mode, monkeypatch):
    from oracle import oracle as orc
    if mode == "async_slices":
        monkeypatch.setenv("MLRA_TEST_ASYNC", "1")  # inherited by the spawned workers
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w, a, b, alpha, x, g = _case()
    _, xb = orc.layer_forward(w, a, b, alpha, None, x)
    _, da, db, dbias = orc.layer_backward(w, a, b, alpha, x, xb, g, need_dx=False, need_dbias=True)
    # fp32 bucket: sums of fp32-rounded shard gradients
    np.testing.assert_allclose(got["l.dA"], da, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(got["l.dB"], db, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(got["l.dbias"], dbias, rtol=1e-5, atol=1e-6)
