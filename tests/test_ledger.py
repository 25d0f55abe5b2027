"""MemoryLedger / ledger_assert_single_materialization (lowprec_linear.hpp:36-80,
lowprec_linear.cpp:62-148), re-expressing the reference's ledger tests
(test_lowprec.cpp:155-320) — the synthetic replay cases verbatim on the CPU,
the recorded-pass cases on the device with device byte counts (SURVEY §8(b)
"Ledger semantics": the weight strategy charges the bf16 Ŵ, the fused
strategies nothing)."""
import numpy as np
import pytest
import torch

from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import modulora as M
from paper_2309_16119_b200.ledger import (LayerDims, MemoryLedger, Phase,
                                          ledger_assert_single_materialization)

S = M.MaterializationStrategy


def test_ledger_replay_arithmetic_on_synthetic_event_streams():
    # test_lowprec.cpp:180-262
    dims = [LayerDims("a", 8, 8), LayerDims("b", 4, 4)]
    good = MemoryLedger()
    good.on_alloc("a", Phase.Forward, 512)
    good.on_free("a", Phase.Forward, 512)
    good.on_alloc("b", Phase.Forward, 128)
    good.on_free("b", Phase.Forward, 128)
    assert good.peak_bytes() == 512 and good.current_bytes() == 0
    ok = ledger_assert_single_materialization(good, dims, S.WeightMaterialize)
    assert ok.passed and ok.observed_peak == 512 and ok.expected_peak == 512
    assert ok.sum_of_layers == (8 * 8 + 4 * 4) * 8 and not ok.violations

    overlap = MemoryLedger()
    overlap.on_alloc("a", Phase.Forward, 512)
    overlap.on_alloc("b", Phase.Forward, 128)
    overlap.on_free("b", Phase.Forward, 128)
    overlap.on_free("a", Phase.Forward, 512)
    bad = ledger_assert_single_materialization(overlap, dims, S.WeightMaterialize)
    assert not bad.passed
    assert any("while another buffer is live" in v for v in bad.violations)

    twin = [LayerDims("a", 8, 8), LayerDims("b", 8, 8)]
    summed = MemoryLedger()
    summed.on_alloc("a", Phase.Forward, 512)
    summed.on_alloc("b", Phase.Forward, 512)
    summed.on_free("a", Phase.Forward, 512)
    summed.on_free("b", Phase.Forward, 512)
    rep = ledger_assert_single_materialization(summed, twin, S.WeightMaterialize)
    assert not rep.passed and any("peak equals the sum over layers" in v for v in rep.violations)

    leak = MemoryLedger()
    leak.on_alloc("a", Phase.Forward, 512)
    assert not ledger_assert_single_materialization(leak, dims, S.WeightMaterialize).passed

    empty = MemoryLedger()
    assert not ledger_assert_single_materialization(empty, dims, S.WeightMaterialize).passed
    em = ledger_assert_single_materialization(empty, dims, S.QuantizerMatvec)
    assert em.passed and em.expected_peak == 0

    rows = [LayerDims("a", 2, 4), LayerDims("b", 2, 16)]
    row_led = MemoryLedger()
    row_led.on_alloc("a", Phase.Forward, 32)
    row_led.on_free("a", Phase.Forward, 32)
    row_led.on_alloc("b", Phase.Forward, 128)
    row_led.on_free("b", Phase.Forward, 128)
    rr = ledger_assert_single_materialization(row_led, rows, S.RowMaterialize)
    assert rr.passed and rr.expected_peak == 128

    broken = MemoryLedger()
    with pytest.raises(MlraError) as e:
        broken.on_free("a", Phase.Forward, 64)
    assert e.value.status == 5  # ContractError


def test_device_dims_change_the_empty_rule():
    # a fused device pass materializes nothing: no events is the correct record
    dims = [LayerDims("a", 256, 512, device_bytes=0)]
    assert ledger_assert_single_materialization(MemoryLedger(), dims, S.RowMaterialize).passed


def _layers(strategy):
    from tests.gpu_util import random_quantized
    out = []
    for i, (rows, cols) in enumerate([(256, 512), (512, 768), (384, 256)]):
        dq = M.DeviceQuantizedMatrix(random_quantized(rows, cols, 3, 128, 900 + i)[0])
        a = torch.randn(rows, 8, device="cuda") * 0.02
        b = torch.randn(cols, 8, device="cuda") * 0.02
        out.append(M.ModuLoraLayer(f"l{i}", dq, M.LoraAdapter(a, b, 8, 16.0), strategy=strategy))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", list(S))
def test_stacked_layers_materialize_one_buffer_at_a_time(strategy):
    # test_lowprec.cpp:264-310: forward l0, l1, l2 then backward l2, l1, l0
    layers = _layers(strategy)
    led = MemoryLedger()
    m = 64
    xs = [torch.randn(m, L.d_in(), device="cuda").to(torch.bfloat16) for L in layers]
    outs = [M.layer_forward(L, x, ledger=led) for L, x in zip(layers, xs)]
    for L, x, (y, xb) in reversed(list(zip(layers, xs, outs))):
        dy = torch.randn(m, L.d_out(), device="cuda").to(torch.bfloat16)
        M.layer_backward(L, x, xb, dy, ledger=led)
    torch.cuda.synchronize()
    dims = [LayerDims.of(M.LpLinearContext(L.weights, strategy, L.name)) for L in layers]
    rep = ledger_assert_single_materialization(led, dims, strategy)
    assert rep.passed, rep.violations
    assert led.current_bytes() == 0
    if strategy == S.WeightMaterialize:
        ev = led.events()
        assert len(ev) == 12
        order = ["l0", "l0", "l1", "l1", "l2", "l2", "l2", "l2", "l1", "l1", "l0", "l0"]
        assert [e.layer for e in ev] == order
        assert [e.phase for e in ev] == [Phase.Forward] * 6 + [Phase.Backward] * 6
        assert [e.alloc for e in ev] == [True, False] * 6
        assert led.peak_bytes() == max(L.d_out() * L.d_in() for L in layers) * 2
    else:  # fused: Ŵ never exists in HBM
        assert led.events() == [] and rep.expected_peak == 0


@pytest.mark.gpu
def test_lp_forward_backward_charge_the_ledger():
    # test_lowprec.cpp:155-178: one context, forward + backward, 4 events
    from tests.gpu_util import random_quantized
    dq = M.DeviceQuantizedMatrix(random_quantized(256, 512, 4, 128, 77)[0])
    led = MemoryLedger()
    ctx = M.LpLinearContext(dq, S.WeightMaterialize, "solo", None, led)
    x = torch.randn(32, 512, device="cuda").to(torch.bfloat16)
    g = torch.randn(32, 256, device="cuda").to(torch.bfloat16)
    M.lp_forward(ctx, x)
    M.lp_backward(ctx, g)
    assert led.current_bytes() == 0 and led.peak_bytes() == 256 * 512 * 2
    ev = led.events()
    assert len(ev) == 4 and ev[0].phase == Phase.Forward and ev[0].alloc
    assert ev[2].phase == Phase.Backward and ev[2].alloc


@pytest.mark.gpu
def test_quantized_matvec_and_lp_linear_function():
    # quantize.cpp:268-300 (one vector) and the LpLinearFunction tape node
    # (lowprec_linear.cpp:249-266) against the f64 oracle on the same bf16 operands
    from oracle import oracle as orc
    from tests.gpu_util import random_quantized
    q, words, scales, zeros = random_quantized(300, 520, 3, 40, 55)
    dq = M.DeviceQuantizedMatrix(q)
    w = orc.bf16_round(orc.dequantize(words, 300, 520, 3, 40, scales, zeros))
    v = orc.bf16_round(orc.gaussian(56, 1, 520))[0]
    u = orc.bf16_round(orc.gaussian(57, 1, 300))[0]
    y = M.quantized_matvec(dq, torch.from_numpy(v).cuda()).double().cpu().numpy()
    yt = M.quantized_matvec_transposed(dq, torch.from_numpy(u).cuda()).double().cpu().numpy()
    assert np.linalg.norm(y - w @ v) <= 1e-5 * np.linalg.norm(w @ v)
    assert np.linalg.norm(yt - w.T @ u) <= 1e-5 * np.linalg.norm(w.T @ u)
    x = torch.from_numpy(orc.bf16_round(orc.gaussian(58, 7, 520))).float().cuda().requires_grad_(True)
    out = M.LpLinearFunction.apply(x, M.LpLinearContext(dq, S.RowMaterialize, "lp"))
    g = torch.from_numpy(orc.bf16_round(orc.gaussian(59, 7, 300))).float().cuda()
    out.backward(g)
    xr = x.detach().double().cpu().numpy()
    assert np.linalg.norm(out.detach().double().cpu().numpy() - xr @ w.T) <= 1e-5 * np.linalg.norm(xr @ w.T)
    gd = g.double().cpu().numpy()
    assert np.linalg.norm(x.grad.double().cpu().numpy() - gd @ w) <= 1e-5 * np.linalg.norm(gd @ w)
