"""Data-parallel TransformerTrainer (model.py): two ranks, each with half of
the batch, all-reduce their per-layer gradient spans during the backward and
scale by 1/world — the gradients must equal the one-process full-batch ones
(up to the summation order of dA / dB over tokens, which the split changes).

The box has one GPU, so both ranks share cuda:0 and the exchange runs over
gloo (NCCL refuses two ranks on one device); the exchange code path is the
same `dist.all_reduce(async_op=True)` the NCCL run takes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build():
    import json
    from paper_2309_16119_b200 import model as Mdl
    from paper_2309_16119_b200 import train as T
    from paper_2309_16119_b200.checkpoint import Checkpoint
    ck = Checkpoint.load(os.path.join(GOLDEN, "parity_b4_adapted.mlra"))
    model = Mdl.ParityTransformer(ck.to_layers(), json.loads(ck.config_json())["ln_eps"])
    return Mdl.TransformerTrainer(model, T.TrainConfig(lr=1e-2))


def _batch():
    z = np.load(os.path.join(GOLDEN, "parity_model.npz"))
    return torch.from_numpy(z["xs"].astype(np.float32)), torch.from_numpy(z["labels"])


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = _build()
        x, y = _batch()
        per = x.shape[0] // world
        sl = slice(rank * per, (rank + 1) * per)
        loss = tr.loss_and_grads(x[sl].cuda(), y[sl].cuda())
        torch.cuda.synchronize()
        if rank == 0:
            np.save(out_path, tr.grads.flat.double().cpu().numpy())
        tr.step(x[sl].cuda(), y[sl].cuda())  # a full step (AdamW) runs under DP too
        flat = tr.params.flat.detach().cpu().clone()
        torch.cuda.synchronize()
        gathered = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(gathered, flat)
        assert torch.equal(gathered[0], gathered[1]), "replicas diverged after a DP step"
        assert torch.isfinite(loss)
    finally:
        dist.destroy_process_group()


def test_transformer_trainer_two_ranks_match_full_batch(tmp_path):
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    g2 = np.load(out)
    tr = _build()
    x, y = _batch()
    tr.loss_and_grads(x.cuda(), y.cuda())
    g1 = tr.grads.flat.double().cpu().numpy()
    assert np.linalg.norm(g2 - g1) <= 1e-3 * np.linalg.norm(g1)
