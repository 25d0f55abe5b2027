"""The .mlra checkpoint -> device path.

Fixtures (tests/golden/*.mlra, checkpoints.json) come from the reference
itself (tests/golden/make_golden.py: the CLI `quantize` recipe through
oracle/_ref, then the reference's own load_model on corrupted variants). The
first one is the reference's golden.mlra: its file and frozen-state digests
are the constants pinned in acceptance.cpp:462-463 / test_checkpoint.cpp:31-32.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200.checkpoint import Checkpoint, inspect_layout, load_model
from tests.golden.make_golden import CKPTS, corruptions

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EXPECT = json.load(open(os.path.join(GOLDEN, "checkpoints.json")))
NAMES = [c[0] for c in CKPTS]


def test_golden_digests_pinned():
    c = load_model(os.path.join(GOLDEN, "golden.mlra"))
    assert c.file_hash() == 0xb48207d130703ee4
    assert c.frozen_hash() == 0xa3d66a9e729158ff


@pytest.mark.parametrize("name", NAMES)
def test_load_save_byte_identical(name, tmp_path):
    path = os.path.join(GOLDEN, name)
    c = Checkpoint.load(path)
    assert c.file_hash() == EXPECT[name]["file_hash"]
    assert c.frozen_hash() == EXPECT[name]["frozen_hash"]
    out = str(tmp_path / "copy.mlra")
    c.save(out)
    assert open(out, "rb").read() == open(path, "rb").read()


@pytest.mark.parametrize("name", NAMES)
def test_corrupt_files_match_reference_errors(name, tmp_path):
    buf = open(os.path.join(GOLDEN, name), "rb").read()
    for cname, data in corruptions(buf).items():
        want = EXPECT[f"{name}:{cname}"]
        p = str(tmp_path / "c.mlra")
        with open(p, "wb") as fh:
            fh.write(data)
        if want["status"] == 0:
            c = Checkpoint.load(p)
            assert c.file_hash() == want["file_hash"] and c.frozen_hash() == want["frozen_hash"]
            continue
        with pytest.raises(MlraError) as e:
            Checkpoint.load(p)
        assert e.value.status == want["status"], cname
        assert e.value.format_kind == ["BadMagic", "BadVersion", "Truncated", "BadField"][want["format_kind"]], cname
        assert e.value.offset == want["offset"], cname


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(MlraError) as e:
        Checkpoint.load(str(tmp_path / "nope.mlra"))
    assert e.value.kind == "IoError"


def test_records_decode_like_the_oracle():
    c = Checkpoint.load(os.path.join(GOLDEN, "parity_b4.mlra"))
    lay = inspect_layout(os.path.join(GOLDEN, "parity_b4.mlra"))
    assert len(lay["layers"]) == len(c) == 7 and lay["version"] == 1
    for i in range(len(c)):
        r = c.layer(i)
        assert orc._Lib.get().orc_validate_qmatrix(
            r.rows, r.cols, r.bits, r.bits, r.group_size, r.rows * r.cols, r.scales.size,
            r.zeros.size, r.scales) == 0
        assert orc._Lib.get().orc_validate_packed(r.words, r.words.size, r.rows * r.cols, r.bits) == 0
        assert r.a.shape == (r.rows, r.rank) and r.b.shape == (r.cols, r.rank)
        assert r.bias.shape == (r.rows,)


def test_set_adapter_rewrites_only_adapter_section(tmp_path):
    path = os.path.join(GOLDEN, "golden.mlra")
    c = Checkpoint.load(path)
    r = c.layer(0)
    c.set_adapter(0, r.a + 1.0, r.b * 0.5)
    out = str(tmp_path / "ft.mlra")
    c.save(out)
    a0, a1 = open(path, "rb").read(), open(out, "rb").read()
    assert len(a0) == len(a1)
    diff = np.nonzero(np.frombuffer(a0, np.uint8) != np.frombuffer(a1, np.uint8))[0]
    assert diff.min() >= r.adapter_offset and diff.max() < r.adapter_offset + r.adapter_size
    c2 = Checkpoint.load(out)
    assert c2.frozen_hash() == c.frozen_hash()
    assert np.array_equal(c2.layer(0).a, r.a + 1.0)
    with pytest.raises(MlraError):
        c.set_adapter(0, r.a[:1], r.b)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_upload_verbatim_and_materialize_bit_exact(name):
    c = Checkpoint.load(os.path.join(GOLDEN, name))
    for i in range(len(c)):
        r = c.layer(i)
        dq = c.upload(i)
        want = orc.dequantize_f32(r.words, r.rows, r.cols, r.bits, r.group_size, r.scales, r.zeros)
        got = __import__("paper_2309_16119_b200").dequantize(dq, torch.float32).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
def test_checkpoint_layers_run_forward_backward():
    from paper_2309_16119_b200 import modulora as M
    c = Checkpoint.load(os.path.join(GOLDEN, "parity_b4.mlra"))
    layers = c.to_layers()
    for i, L in enumerate(layers):
        r = c.layer(i)
        x64 = orc.bf16_round(orc.gaussian(90 + i, 37, r.cols))
        x = torch.from_numpy(x64.astype(np.float32)).to(torch.bfloat16).cuda()
        y, xb = M.layer_forward(L, x, out_dtype=torch.float32)
        w = orc.dequantize(r.words, r.rows, r.cols, r.bits, r.group_size, r.scales, r.zeros)
        a32 = r.a.astype(np.float32).astype(np.float64)
        b32 = r.b.astype(np.float32).astype(np.float64)
        yr, _ = orc.layer_forward(w, a32, b32, r.alpha, r.bias.astype(np.float64), x64)
        assert np.linalg.norm(y.double().cpu().numpy() - yr) <= 4e-3 * np.linalg.norm(yr) + 1e-6


STRUCT = ["dup_last_adapter", "missing_last_adapter", "no_adapters", "swapped_adapters",
          "dup_first_for_second", "alpha_zero", "alpha_negative"]


@pytest.mark.parametrize("name", NAMES)
def test_assemble_model_checks_match_reference(name, tmp_path):
    """adapter sections the reference's load_model rejects in
    assemble_model (model.cpp:472-531: one adapter per layer, in layer order,
    rank >= 1, alpha > 0) are rejected by load_model with the same ConfigError;
    the parse alone (inspect_layout) still accepts them, keeps every record in
    file order and re-encodes byte-identically."""
    from tests.golden.make_golden import record_offsets, structural_corruptions
    buf = open(os.path.join(GOLDEN, name), "rb").read()
    for cname, data in structural_corruptions(buf).items():
        want = EXPECT[f"{name}:{cname}"]
        p = str(tmp_path / "s.mlra")
        with open(p, "wb") as fh:
            fh.write(data)
        c = Checkpoint.load(p)
        assert [a[:3] for a in record_offsets(data)[2]] == c.layout()["adapters"], cname
        out = str(tmp_path / "s2.mlra")
        c.save(out)
        assert open(out, "rb").read() == data, cname
        if want["status"] == 0:
            assert load_model(p).frozen_hash() == want["frozen_hash"]
            continue
        with pytest.raises(MlraError) as e:
            load_model(p)
        assert e.value.status == want["status"] and e.value.kind == "ConfigError", cname


def test_to_layers_follows_the_config(tmp_path):
    """to_layers() takes strategy and bias_trainable from the config JSON
    (assemble_model, model.cpp:527-529) unless the caller overrides them."""
    import paper_2309_16119_b200.checkpoint as CK
    c = Checkpoint.load(os.path.join(GOLDEN, "parity_b4.mlra"))
    cfg = c.config()
    assert "strategy" in cfg and "bias_trainable" in cfg
    seen = {}

    class Probe(CK.Checkpoint):
        def upload(self, i, stream=None):
            return None

    orig_torch = CK.torch

    class _T:  # no GPU here: keep the factors on the host
        def __getattr__(self, k):
            return getattr(orig_torch, k)

        @staticmethod
        def from_numpy(a):
            class _W:
                def __init__(self, t):
                    self.t = t

                def cuda(self):
                    return self.t
            return _W(orig_torch.from_numpy(a))
    CK.torch = _T()
    try:
        p = Probe(c._h)
        c._h = None
        layers = p.to_layers()
        seen["strategy"] = {int(L.strategy) for L in layers}
        seen["bias"] = {L.bias_trainable for L in layers}
        forced = p.to_layers(bias_trainable=True)
        assert all(L.bias_trainable for L in forced)
    finally:
        CK.torch = orig_torch
    from paper_2309_16119_b200.modulora import parse_strategy
    assert seen["strategy"] == {int(parse_strategy(cfg["strategy"]))}
    assert seen["bias"] == {bool(cfg["bias_trainable"])}
