"""Pin the C oracle (oracle/mlra_oracle.c) to the reference's own answers.

Fixtures in tests/golden/ were produced by the unmodified reference
(tests/golden/make_golden.py). Everything here is bit-exact: the oracle
restates the reference's f64 evaluation order.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import load_golden


def test_rng_stream_matches_reference():
    g = load_golden("rng.npz")
    assert np.array_equal(orc.gaussian(7, 3, 5), g["gaussian_seed7"])
    assert np.array_equal(orc.gaussian(8, 4, 4, 0.5, 0.02), g["gaussian_seed8_scaled"])
    assert orc.mix_seed(11, 0xADA9) == int(g["mix_seed_11_ada9"][0])


def test_frozen_word_layout(golden_bitpack):
    # test_bitpack.cpp:29-37
    w = orc.pack([3, 1, 2, 0], 2)
    assert w.tolist() == [0x27]
    assert np.array_equal(w, golden_bitpack["kat_words_3120_b2"])


def test_word_counts():
    # test_bitpack.cpp:39-49
    assert orc.packed_word_count(4, 2) == 1
    assert orc.packed_word_count(11, 3) == 2
    assert orc.packed_word_count(32, 8) == 8
    assert orc.packed_word_count(0, 4) == 0
    assert orc.packed_word_count(16, 2) == 1
    assert orc.packed_word_count(17, 2) == 2


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 5, 31, 32, 33, 64, 100, 200])
def test_roundtrip_matches_reference_words(golden_bitpack, bits, n):
    codes = golden_bitpack[f"rt_b{bits}_n{n}_codes"]
    words = orc.pack(codes, bits)
    assert np.array_equal(words, golden_bitpack[f"rt_b{bits}_n{n}_words"])
    assert np.array_equal(orc.unpack(words, n, bits), codes)


def test_corrupted_and_out_of_range(golden_bitpack):
    # test_bitpack.cpp:102-124
    codes = golden_bitpack["rows7x9_codes"][:11]
    w = orc.pack(codes, 3)
    with pytest.raises(RuntimeError):
        orc.unpack(np.append(w, 0), 11, 3)
    with pytest.raises(RuntimeError):
        orc.unpack(w[:-1], 11, 3)
    bad = w.copy()
    bad[-1] |= 0x80000000
    with pytest.raises(RuntimeError):
        orc.unpack(bad, 11, 3)
    with pytest.raises(IndexError):
        orc.pack([4], 2)
    with pytest.raises(IndexError):
        orc.pack([0, 1, 8], 3)
    with pytest.raises(ValueError):
        orc.pack([0], 5)


def _qcases(golden_quant):
    i = 0
    while f"q{i}_meta" in golden_quant:
        yield i
        i += 1


def test_dequant_hand_example(golden_quant):
    # test_quantize.cpp:34-60
    rows, cols, bits, g = golden_quant["q0_meta"]
    deq = orc.dequantize(golden_quant["q0_words"], rows, cols, bits, g,
                         golden_quant["q0_scales"], golden_quant["q0_zeros"])
    assert deq.tolist() == [[-1.0, -0.5], [2.0, 3.0]]
    assert np.array_equal(deq, golden_quant["q0_deq"])


def test_rtn_and_dequant_bit_exact(golden_quant):
    n = 0
    for i in _qcases(golden_quant):
        if f"q{i}_w" not in golden_quant:
            continue
        rows, cols, bits, g = (int(v) for v in golden_quant[f"q{i}_meta"])
        words, scales, zeros = orc.quantize_rtn(golden_quant[f"q{i}_w"], bits, g)
        assert np.array_equal(words, golden_quant[f"q{i}_words"]), i
        assert np.array_equal(scales, golden_quant[f"q{i}_scales"]), i
        assert np.array_equal(zeros, golden_quant[f"q{i}_zeros"]), i
        deq = orc.dequantize(words, rows, cols, bits, g, scales, zeros)
        assert np.array_equal(deq, golden_quant[f"q{i}_deq"]), i
        # materialize contract: f32 image is RN of the f64 value
        f32 = orc.dequantize_f32(words, rows, cols, bits, g, scales, zeros)
        assert np.array_equal(f32, golden_quant[f"q{i}_deq"].astype(np.float32)), i
        n += 1
    assert n >= 8


def _lcases(golden_layer):
    i = 0
    while f"l{i}_meta" in golden_layer:
        yield i
        i += 1


def test_layer_forward_backward_bit_exact(golden_layer):
    n = 0
    for i in _lcases(golden_layer):
        p = f"l{i}_"
        d_out, d_in, bits, g, r, m, has_bias, need_dx = (int(v) for v in golden_layer[p + "meta"])
        alpha = float(golden_layer[p + "alpha"][0])
        w = orc.dequantize(golden_layer[p + "words"], d_out, d_in, bits, g,
                           golden_layer[p + "scales"], golden_layer[p + "zeros"])
        bias = golden_layer[p + "bias"] if has_bias else None
        y, xb = orc.layer_forward(w, golden_layer[p + "a"], golden_layer[p + "b"], alpha, bias,
                                  golden_layer[p + "x"])
        assert np.array_equal(y, golden_layer[p + "y"]), i
        dx, da, db, dbias = orc.layer_backward(w, golden_layer[p + "a"], golden_layer[p + "b"],
                                               alpha, golden_layer[p + "x"], xb,
                                               golden_layer[p + "g"], need_dx=bool(need_dx),
                                               need_dbias=bool(has_bias))
        assert np.array_equal(da, golden_layer[p + "da"]), i
        assert np.array_equal(db, golden_layer[p + "db"]), i
        if need_dx:
            assert np.array_equal(dx, golden_layer[p + "dx"]), i
        if has_bias:
            assert np.array_equal(dbias, golden_layer[p + "dbias"]), i
        n += 1
    assert n == 6


def test_identity_passes_through():
    # test_lowprec.cpp:73-82: make_identity_quantized(6), 8-bit, s=1, z=0
    n = 6
    codes = np.eye(n, dtype=np.uint32).ravel()
    words = orc.pack(codes, 8)
    w = orc.dequantize(words, n, n, 8, n, np.ones(n, np.float32), np.zeros(n, np.float32))
    x = orc.gaussian(1, 3, 6)
    g = orc.gaussian(2, 3, 6)
    assert np.array_equal(orc.lp_forward(w, x), x)
    assert np.array_equal(orc.lp_backward(w, g), g)
