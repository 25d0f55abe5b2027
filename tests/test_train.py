"""The adapter optimizer on the device and the stack training step (SURVEY
§8(f)2). The oracle's AdamW (oracle/mlra_oracle.c orc_adamw_step, a
restatement of train.cpp:81-134) is pinned bit-for-bit against the reference
itself (oracle/_ref: the reference's own AdamW class) and its known-answer
test (test_train.cpp:145-167); the device kernel is then checked bit-for-bit
against the oracle."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import train as T

_have_ref = orc.Ref.available()


def _problem(sizes, steps, seed, bad=None):
    rng = np.random.default_rng(seed)
    total = sum(sizes)
    values = rng.normal(0, 0.5, total)
    grads = rng.normal(0, 0.1, (steps, total)) * np.exp(rng.normal(0, 2, (steps, total)))
    if bad is not None:
        s, j = bad
        grads[s, j] = np.inf if j % 2 else np.nan
    lrs = np.array([1e-2 * (1 + 0.1 * k) for k in range(steps)])
    return values, grads, lrs


def _oracle_run(sizes, values, grads, lrs, **kw):
    offs = np.cumsum([0] + list(sizes))
    ps = [values[offs[i]:offs[i + 1]].copy() for i in range(len(sizes))]
    ms = [np.zeros(s) for s in sizes]
    vs = [np.zeros(s) for s in sizes]
    for s, lr in enumerate(lrs):
        gs = [grads[s, offs[i]:offs[i + 1]] for i in range(len(sizes))]
        first = orc.adamw_step(ps, ms, vs, gs, s, lr, **kw)
        if first < len(sizes):
            return np.concatenate(ps), s, first
    return np.concatenate(ps), None, None


# ----------------------------------------------------------------------------- CPU
def test_oracle_adamw_known_answer():
    # test_train.cpp:145-167
    p = [np.array([1.0, -2.0, 3.0])]
    g = [np.array([0.1, -0.2, 0.3])]
    m, v = [np.zeros(3)], [np.zeros(3)]
    assert orc.adamw_step(p, m, v, g, 0, 0.01, 0.9, 0.999, 1e-8, 0.0) == 1
    for j in range(3):
        gj = g[0][j]
        mm = (1.0 - 0.9) * gj
        vv = (1.0 - 0.999) * gj * gj
        mhat = mm / (1.0 - math.pow(0.9, 1.0))
        vhat = vv / (1.0 - math.pow(0.999, 1.0))
        want = [1.0, -2.0, 3.0][j] * (1.0 - 0.01 * 0.0) - 0.01 * mhat / (math.sqrt(vhat) + 1e-8)
        assert p[0][j] == want


@pytest.mark.skipif(not _have_ref, reason="reference library not built")
@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_oracle_adamw_matches_reference_bitwise(wd):
    sizes = [7, 130, 1, 64]
    values, grads, lrs = _problem(sizes, 12, seed=5)
    rc, ref_vals, _ = orc.Ref.adamw_run(sizes, values, grads, lrs, wd=wd)
    assert rc == 0
    got, _, _ = _oracle_run(sizes, values, grads, lrs, weight_decay=wd)
    assert np.array_equal(got.view(np.uint64), ref_vals.view(np.uint64))


@pytest.mark.skipif(not _have_ref, reason="reference library not built")
def test_oracle_adamw_nonfinite_matches_reference():
    sizes = [5, 9, 3]
    values, grads, lrs = _problem(sizes, 4, seed=6, bad=(2, 7))  # step 2, parameter 1
    rc, ref_vals, bad_step = orc.Ref.adamw_run(sizes, values, grads, lrs)
    assert rc == 6 and bad_step == 2
    got, s, first = _oracle_run(sizes, values, grads, lrs)
    assert (s, first) == (2, 1)
    assert np.array_equal(got.view(np.uint64), ref_vals.view(np.uint64))


def test_lr_schedule_and_config():
    c = T.TrainConfig(steps=10, lr=0.1, warmup_ratio=0.2, schedule=T.LrSchedule.Cosine)
    assert T.lr_at(c, 0) == 0.1 * 1 / 2 and T.lr_at(c, 1) == 0.1
    assert T.lr_at(c, 2) == 0.1 * 0.5 * (1.0 + math.cos(3.14159265358979323846 * 0.0))
    assert T.lr_at(c, 6) == 0.1 * 0.5 * (1.0 + math.cos(3.14159265358979323846 * (4 / 8)))
    c.schedule = T.LrSchedule.Linear
    assert T.lr_at(c, 6) == 0.1 * (1.0 - 4 / 8)
    assert T.parse_schedule("cosine") == T.LrSchedule.Cosine
    with pytest.raises(MlraError):
        T.parse_schedule("step")
    with pytest.raises(MlraError):
        T.TrainConfig(beta1=1.0).validate()


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("gdtype", [torch.float64, torch.float32])
def test_device_adamw_bit_exact(gdtype):
    sizes = [7, 4096, 1, 640, 33]
    values, grads, lrs = _problem(sizes, 6, seed=7)
    if gdtype == torch.float32:
        grads = grads.astype(np.float32).astype(np.float64)
    want, _, _ = _oracle_run(sizes, values, grads, lrs, weight_decay=0.01)
    opt = T.AdamW(0.9, 0.999, 1e-8, 0.01)
    p = torch.from_numpy(values.copy()).cuda()
    names = [f"p{i}" for i in range(len(sizes))]
    for s, lr in enumerate(lrs):
        g = torch.from_numpy(grads[s].copy()).to(gdtype).cuda()
        opt.step(p, sizes, names, g, s, lr)
    got = p.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_device_adamw_nonfinite_semantics():
    sizes = [5, 9, 3]
    values, grads, lrs = _problem(sizes, 4, seed=6, bad=(2, 7))
    want, s_bad, first = _oracle_run(sizes, values, grads, lrs)
    opt = T.AdamW()
    p = torch.from_numpy(values.copy()).cuda()
    names = ["l.A", "l.B", "l.bias"]
    for s, lr in enumerate(lrs):
        g = torch.from_numpy(grads[s].copy()).cuda()
        if s == s_bad:
            with pytest.raises(MlraError) as e:
                opt.step(p, sizes, names, g, s, lr)
            assert e.value.kind == "NumericError" and "'l.B'" in str(e.value)
            break
        opt.step(p, sizes, names, g, s, lr)
    assert np.array_equal(p.cpu().numpy().view(np.uint64), want.view(np.uint64))
    # asynchronous form: the index lands in a device int, nothing raised
    opt2 = T.AdamW()
    p2 = torch.from_numpy(values.copy()).cuda()
    bad = opt2.step(p2, sizes, names, torch.from_numpy(grads[2].copy()).cuda(), 0, 0.01,
                    check_finite=False)
    assert int(bad.item()) == 1


@pytest.mark.gpu
def test_stack_trainer_step_matches_oracle():
    from paper_2309_16119_b200 import modulora as M
    from tests.gpu_util import random_quantized, to_bf16_dev
    shapes = [(512, 256), (256, 512), (768, 256)]
    layers, xs, dys = [], [], []
    for i, (d_out, d_in) in enumerate(shapes):
        q, *_ = random_quantized(d_out, d_in, 3, 128, seed=40 + i)
        L = M.make_layer(f"l{i}", M.DeviceQuantizedMatrix(q), 8, 16.0, seed=50 + i,
                         bias_trainable=(i == 1))
        L.adapter.a = torch.randn(d_out, 8, device="cuda") * 0.02
        layers.append(L)
        xs.append(to_bf16_dev(orc.gaussian(60 + i, 200, d_in)))
        dys.append(to_bf16_dev(orc.gaussian(70 + i, 200, d_out)))
    cfg = T.TrainConfig(steps=3, lr=1e-3, weight_decay=0.01)
    tr = T.LinearStackTrainer(layers, cfg)
    before = tr.params.flat.double().cpu().numpy()
    for step in range(2):
        outs = tr.forward(xs)
        tr.backward(xs, [xb for _, xb in outs], dys)
        grads = tr.grads.flat.double().cpu().numpy()
        # reference arithmetic on the same gradients, from the f64 masters
        if step == 0:
            ps = [before.copy()]
            ms, vs = [np.zeros_like(before)], [np.zeros_like(before)]
        orc.adamw_step(ps, ms, vs, [grads], step, T.lr_at(cfg, step), 0.9, 0.999, 1e-8, 0.01)
        tr.optimizer_step()
        assert np.array_equal(tr.opt.master.cpu().numpy().view(np.uint64), ps[0].view(np.uint64))
        assert np.array_equal(tr.params.flat.cpu().numpy(), ps[0].astype(np.float32))
    # the layers read the updated factors (views into the flat parameter bucket)
    assert layers[0].adapter.a.data_ptr() == tr.params.flat.data_ptr()


@pytest.mark.gpu
def test_stack_trainer_fits_a_planted_adapter():
    # finetune efficacy (the reference's C7, acceptance.cpp): a target made by a
    # planted rank-r update of the frozen layer is fitted by training the adapter
    # with the device step (fwd, bwd, AdamW); the loss must fall by 10x
    from paper_2309_16119_b200 import modulora as M
    from tests.gpu_util import random_quantized
    d_out, d_in, r, m = 256, 512, 8, 512
    q, *_ = random_quantized(d_out, d_in, 4, 128, seed=90)
    L = M.make_layer("l", M.DeviceQuantizedMatrix(q), r, 16.0, seed=91)
    g = torch.Generator(device="cpu").manual_seed(92)
    x = torch.randn(m, d_in, generator=g).cuda().to(torch.bfloat16)
    with torch.no_grad():
        base, _ = M.layer_forward(L, x, out_dtype=torch.float32)
        bp = (torch.randn(d_in, r, generator=g) * 0.05).cuda()
        ap = (torch.randn(d_out, r, generator=g) * 0.05).cuda()
        planted = (x.float() @ bp) @ ap.T  # representable by the adapter: s·(x·B)·Aᵀ
        target = base + planted
    tr = T.LinearStackTrainer([L], T.TrainConfig(steps=200, lr=3e-3))
    losses = []
    for _ in range(200):
        (y, xb), = tr.forward([x])
        diff = y.float() - target
        losses.append(float((diff ** 2).mean()))
        tr.backward([x], [xb], [diff.to(torch.bfloat16)])  # ∝ d(mean sq. error)/dy
        tr.optimizer_step(check_finite=False)
    assert losses[-1] < 0.1 * losses[0], (losses[0], losses[-1])
