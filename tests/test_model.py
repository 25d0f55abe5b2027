"""The decoder-layer caller: the parity transformer of
model.cpp:226-292 on the device (paper_2309_16119_b200/model.py).

Pinned by tests/golden/parity_model.npz: the reference's own model_loss +
tape backward (oracle/ref_driver.cpp ref_parity_loss_grads) on the
reference-made parity_b4.mlra with seeded adapters
(tests/golden/parity_b4_adapted.mlra) and seeded sequences.

CPU: a torch-f64 restatement of the model (test infrastructure: oracle
dequantize + autograd) reproduces the reference's loss and every adapter
gradient to ~1e-12, which pins the glue semantics (norm, attention scale,
pooling, GELU form, loss mean) the device model follows. GPU: the device model
(bf16 operands into the fused kernels, fp32 glue) against the same fixture
within the bf16 tolerance, and a short training run that fits a batch.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200.checkpoint import Checkpoint

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CKPT = os.path.join(GOLDEN, "parity_b4_adapted.mlra")


def _fixture():
    z = np.load(os.path.join(GOLDEN, "parity_model.npz"))
    return z["xs"], z["labels"], float(z["loss"][0]), z["grads"]


def _f64_model_loss(ck: Checkpoint, xs, labels):
    """model.cpp:226-292 restated in torch f64 over the oracle's Ŵ."""
    import torch.nn.functional as F
    eps = json.loads(ck.config_json())["ln_eps"]
    params, lin = [], []
    for i in range(len(ck)):
        r = ck.layer(i)
        w = torch.from_numpy(orc.dequantize(r.words, r.rows, r.cols, r.bits, r.group_size,
                                            r.scales, r.zeros))
        a = torch.from_numpy(r.a.copy()).requires_grad_(True)
        b = torch.from_numpy(r.b.copy()).requires_grad_(True)
        bias = torch.from_numpy(r.bias.astype(np.float64))
        s = r.alpha / r.rank
        params += [a, b]
        lin.append(lambda h, w=w, a=a, b=b, bias=bias, s=s: h @ w.T + s * ((h @ b) @ a.T) + bias)
    x = torch.from_numpy(xs)
    d = x.shape[-1]
    ln1 = F.layer_norm(x, (d,), eps=eps)
    q, k, v = lin[0](ln1), lin[1](ln1), lin[2](ln1)
    sc = (q @ k.transpose(1, 2)) / np.sqrt(float(ck.layer(0).rows))
    h = x + lin[3](torch.softmax(sc, -1) @ v)
    ln2 = F.layer_norm(h, (h.shape[-1],), eps=eps)
    h2 = h + lin[5](F.gelu(lin[4](ln2)))
    logits = lin[6](h2.mean(1))
    loss = F.cross_entropy(logits, torch.from_numpy(labels.astype(np.int64)))
    loss.backward()
    return loss.item(), np.concatenate([p.grad.numpy().ravel() for p in params])


# ----------------------------------------------------------------------------- CPU
def test_fixture_matches_live_reference():
    if not orc.Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    xs, labels, loss, grads = _fixture()
    l2, g2 = orc.Ref.parity_loss_grads(CKPT, xs, labels, grads.size)
    assert l2 == loss and np.array_equal(g2, grads)


def test_f64_restatement_matches_reference():
    xs, labels, loss, grads = _fixture()
    l2, g2 = _f64_model_loss(Checkpoint.load(CKPT), xs, labels)
    assert abs(l2 - loss) <= 1e-12 * abs(loss)
    assert np.max(np.abs(g2 - grads)) <= 1e-11 * np.max(np.abs(grads))


def test_layer_names_and_shapes_enforced():
    from paper_2309_16119_b200.model import ParityTransformer

    class _L:
        def __init__(self, name):
            self.name = name

        def d_in(self):
            return 16

    with pytest.raises(MlraError):
        ParityTransformer([_L("attn_q")] * 6)
    names = ["attn_q", "attn_k", "attn_v", "attn_o", "mlp_in", "mlp_out", "head"]
    with pytest.raises(MlraError):
        ParityTransformer([_L(n) for n in names[:-1]] + [_L("out")])
    with pytest.raises(MlraError):
        ParityTransformer([_L(n) for n in names], ln_eps=0.0)


# ----------------------------------------------------------------------------- GPU
def _device_model():
    from paper_2309_16119_b200 import model as Mdl
    from paper_2309_16119_b200 import train as T
    ck = Checkpoint.load(CKPT)
    eps = json.loads(ck.config_json())["ln_eps"]
    model = Mdl.ParityTransformer(ck.to_layers(), ln_eps=eps)
    return model, Mdl.TransformerTrainer(model, T.TrainConfig(lr=1e-2))


@pytest.mark.gpu
def test_parity_transformer_matches_reference():
    xs, labels, loss, grads = _fixture()
    model, tr = _device_model()
    x = torch.from_numpy(xs.astype(np.float32)).cuda()
    y = torch.from_numpy(labels).cuda()
    got = float(tr.loss_and_grads(x, y))
    g = torch.cat([t.reshape(-1) for t in tr.param_grads()]).double().cpu().numpy()
    assert g.shape == grads.shape
    # bf16 operands into every linear (the kernels' contract), fp32 glue
    assert abs(got - loss) <= 1e-2 * abs(loss)
    assert np.linalg.norm(g - grads) <= 3e-2 * np.linalg.norm(grads)
    # per layer too: no adapter's gradient is lost in the aggregate
    o = 0
    for L in model.layers:
        for n in (L.d_out() * L.adapter.rank, L.d_in() * L.adapter.rank):
            ref = grads[o:o + n]
            assert np.linalg.norm(g[o:o + n] - ref) <= 6e-2 * np.linalg.norm(ref) + 1e-6
            o += n
    # forward only (no trainer): same loss, gradients on the layers
    assert abs(float(model.loss(x, y).detach()) - got) <= 1e-6 * abs(got)


@pytest.mark.gpu
def test_parity_transformer_training_fits_a_batch():
    xs, labels, _, _ = _fixture()
    _, tr = _device_model()
    x = torch.from_numpy(xs.astype(np.float32)).cuda()
    y = torch.from_numpy(labels).cuda()
    losses = [float(tr.step(x, y)) for _ in range(60)]
    assert all(np.isfinite(losses))
    assert losses[-1] < 0.5 * losses[0]
    assert tr.step_index == 60
