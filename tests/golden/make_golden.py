"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference, via oracle/_ref built by
``make -C oracle``):

    python tests/golden/make_golden.py          # everything
    python tests/golden/make_golden.py model    # only parity_model.npz (+ its checkpoint)

Every array is produced by the unmodified reference library
(oracle/_ref/libmlra_ref.so: /root/reference/proj/src + oracle/ref_driver.cpp).
The fixtures pin the C oracle restatement (tests/test_oracle_golden.py) and are
the known answers the GPU parity tests check the CUDA path against. They ship
with the repo, so nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.oracle import Ref  # noqa: E402


def bitpack_cases():
    """test_bitpack.cpp:29-91 known answers."""
    out = {}
    out["kat_words_3120_b2"] = Ref.pack([3, 1, 2, 0], 2)
    for bits in (2, 3, 4, 8):
        for n in (0, 1, 5, 31, 32, 33, 64, 100, 200):
            codes = Ref.random_codes(n, bits, 1000 + n * 10 + bits)  # test_bitpack.cpp:61
            out[f"rt_b{bits}_n{n}_codes"] = codes
            out[f"rt_b{bits}_n{n}_words"] = Ref.pack(codes, bits)
    codes = Ref.random_codes(7 * 9, 3, 5)  # test_bitpack.cpp:78-91 row slices
    out["rows7x9_codes"] = codes
    out["rows7x9_words"] = Ref.pack(codes, 3)
    return out


# (rows, cols, bits, group, seed) — reference-test-like shapes (ragged, not
# row-aligned, e.g. 7x9 at b=3) and LLaMA-aligned tiles (K*b % 128 == 0).
QUANT_CASES = [
    (2, 2, 2, 2, None),       # test_quantize.cpp:34-60 hand example (explicit)
    (7, 9, 3, 3, 101),        # test_lowprec.cpp:98-119 shape, g=3
    (7, 9, 4, 0, 102),
    (16, 32, 2, 4, 103),
    (16, 32, 8, 16, 104),
    (24, 40, 3, 8, 105),
    (64, 256, 4, 128, 106),
    (96, 256, 3, 128, 107),
    (48, 384, 2, 128, 108),
    (32, 128, 8, 64, 109),
]

# (d_out, d_in, bits, group, rank, alpha, m, seed, bias, need_dx)
LAYER_CASES = [
    (7, 9, 3, 3, 2, 8.0, 4, 11, True, True),       # test_lora.cpp:123-150 shape
    (6, 8, 4, 0, 2, 4.0, 3, 12, True, True),       # test_lora.cpp:152-201 shape
    (24, 40, 2, 8, 4, 8.0, 5, 13, False, True),
    (64, 128, 4, 32, 8, 32.0, 16, 14, True, False),   # dx skipped (autodiff.cpp:136)
    (96, 256, 3, 128, 16, 32.0, 20, 15, True, True),
    (256, 128, 4, 128, 8, 16.0, 12, 16, False, True),
]


def quant_cases():
    out = {}
    for i, (rows, cols, bits, group, seed) in enumerate(QUANT_CASES):
        if seed is None:
            from oracle.oracle import Ref as R
            words = R.pack([0, 1, 2, 3], 2)
            scales = np.array([0.5, 1.0], np.float32)
            zeros = np.array([-1.0, 0.0], np.float32)
            g = 2
        else:
            w = Ref.gaussian(seed, rows, cols, 0.0, 0.02 if i % 2 else 1.0)
            words, scales, zeros = Ref.quantize_rtn(w, bits, group)
            g = cols if group == 0 else group
            out[f"q{i}_w"] = w
        deq = Ref.dequantize(words, rows, cols, bits, g, scales, zeros)
        out[f"q{i}_meta"] = np.array([rows, cols, bits, g], np.int64)
        out[f"q{i}_words"] = words
        out[f"q{i}_scales"] = scales
        out[f"q{i}_zeros"] = zeros
        out[f"q{i}_deq"] = deq
    return out


def layer_cases():
    out = {}
    for i, (d_out, d_in, bits, group, r, alpha, m, seed, bias, need_dx) in enumerate(LAYER_CASES):
        w = Ref.gaussian(seed, d_out, d_in, 0.0, 0.02)
        words, scales, zeros = Ref.quantize_rtn(w, bits, group)
        g = d_in if group == 0 else group
        b = np.empty((d_in, r))
        Ref.get().ref_init_adapter_b(d_in, d_out, r, alpha, seed + 1, b)
        a = Ref.gaussian(seed + 2, d_out, r, 0.0, 0.5)  # off its zero init (acceptance.cpp:116-117)
        bvec = Ref.gaussian(seed + 3, 1, d_out, 0.0, 0.3) if bias else None
        x = Ref.gaussian(seed + 4, m, d_in)
        G = Ref.gaussian(seed + 5, m, d_out)
        y, dx, da, db, dbias = Ref.layer_fwd_bwd(words, d_out, d_in, bits, g, scales, zeros,
                                                 a, b, alpha, bvec, x, G, need_dx=need_dx,
                                                 need_dbias=bias)
        p = f"l{i}_"
        out[p + "meta"] = np.array([d_out, d_in, bits, g, r, m, int(bias), int(need_dx)], np.int64)
        out[p + "alpha"] = np.array([alpha])
        out[p + "words"] = words
        out[p + "scales"] = scales
        out[p + "zeros"] = zeros
        out[p + "a"] = a
        out[p + "b"] = b
        if bias:
            out[p + "bias"] = bvec.ravel()
            out[p + "dbias"] = dbias
        out[p + "x"] = x
        out[p + "g"] = G
        out[p + "y"] = y
        if need_dx:
            out[p + "dx"] = dx
        out[p + "da"] = da
        out[p + "db"] = db
    return out


# --------------------------------------------------------------------------- checkpoints
CKPTS = [  # (file, task, bits, seed, group): the first is the reference's own golden.mlra
    ("golden.mlra", "regression", 3, 11, 0),   # test_checkpoint.cpp:28 recipe
    ("parity_b4.mlra", "parity", 4, 5, 0),
    ("regression_b2_g4.mlra", "regression", 2, 7, 4),
    ("regression_b8.mlra", "regression", 8, 9, 0),
]


def field_offsets(buf: bytes) -> dict:
    """Byte offsets of the first layer's fields in a checkpoint (checkpoint.hpp:4-24)."""
    import struct
    o = 6
    (clen,) = struct.unpack_from("<I", buf, o)
    o += 4 + clen
    f = {"n_layers": o}
    o += 4
    f["layer0"] = o
    (nlen,) = struct.unpack_from("<I", buf, o)
    o += 4 + nlen
    rows, cols = struct.unpack_from("<II", buf, o)
    f["rows"], f["cols"] = o, o + 4
    o += 8
    bits = buf[o]
    f["bits"] = o
    o += 1
    (group,) = struct.unpack_from("<I", buf, o)
    f["group"] = o
    o += 4
    f["n_words"] = o
    (nw,) = struct.unpack_from("<I", buf, o)
    o += 4
    f["words"] = o
    f["last_word"] = o + 4 * (nw - 1)
    o += 4 * nw
    ng = rows * (cols // group)
    f["scales"] = o
    o += 8 * ng
    f["bias_len"] = o
    return f


def corruptions(buf: bytes):
    """Deterministic corrupt variants of a checkpoint: name -> bytes."""
    import struct
    f = field_offsets(buf)
    out = {}

    def put(name, off, data):
        b = bytearray(buf)
        b[off:off + len(data)] = data
        out[name] = bytes(b)

    put("bad_magic", 0, b"MLRB")
    put("bad_version", 4, struct.pack("<H", 2))
    put("bits5", f["bits"], bytes([5]))
    put("group7", f["group"], struct.pack("<I", 7))
    put("zero_rows", f["rows"], struct.pack("<I", 0))
    put("word_count", f["n_words"], struct.pack("<I", struct.unpack_from("<I", buf, f["n_words"])[0] + 1))
    put("neg_scale", f["scales"], struct.pack("<f", -1.0))
    put("bias_len", f["bias_len"], struct.pack("<I", 1))
    put("n_layers_big", f["n_layers"], struct.pack("<I", 7))
    out["trailing"] = buf + b"\0"
    for cut in (3, 5, 9, f["layer0"] + 2, f["words"] + 6, f["scales"] + 3, len(buf) - 1):
        out[f"trunc{cut}"] = buf[:cut]
    # nonzero trailing bits: set the top bit of the last packed word when it is padding
    lw = struct.unpack_from("<I", buf, f["last_word"])[0]
    put("trailing_bits", f["last_word"], struct.pack("<I", lw | 0x80000000))
    return out


def record_offsets(buf: bytes):
    """Walk a checkpoint (checkpoint.hpp:4-24): layer records [(name, off, size)],
    the adapter-count offset, adapter records [(name, off, size, alpha_off)]."""
    import struct
    o = 6
    (clen,) = struct.unpack_from("<I", buf, o)
    o += 4 + clen
    (nl,) = struct.unpack_from("<I", buf, o)
    o += 4
    layers, dims = [], {}
    for _ in range(nl):
        off = o
        (n,) = struct.unpack_from("<I", buf, o)
        name = buf[o + 4:o + 4 + n].decode()
        o += 4 + n
        rows, cols = struct.unpack_from("<II", buf, o)
        o += 9
        (group,) = struct.unpack_from("<I", buf, o)
        o += 4
        (nw,) = struct.unpack_from("<I", buf, o)
        o += 4 + 4 * nw + 8 * rows * (cols // group)
        (nb,) = struct.unpack_from("<I", buf, o)
        o += 4 + 4 * nb
        layers.append((name, off, o - off))
        dims[name] = (rows, cols)
    n_ad_off = o
    (na,) = struct.unpack_from("<I", buf, o)
    o += 4
    ads = []
    for _ in range(na):
        off = o
        (n,) = struct.unpack_from("<I", buf, o)
        name = buf[o + 4:o + 4 + n].decode()
        o += 4 + n
        (r,) = struct.unpack_from("<I", buf, o)
        alpha_off = o + 4
        rows, cols = dims[name]
        o += 8 + 8 * r * (rows + cols)
        ads.append((name, off, o - off, alpha_off))
    return layers, n_ad_off, ads


def structural_corruptions(buf: bytes):
    """Well-formed files whose adapter section load_model's assemble_model rejects
    (model.cpp:472-531) or accepts: name -> bytes."""
    import struct
    layers, n_ad_off, ads = record_offsets(buf)
    head, tail = buf[:n_ad_off], buf[n_ad_off + 4:]
    recs = [buf[a[1]:a[1] + a[2]] for a in ads]

    def with_recs(rs):
        return head + struct.pack("<I", len(rs)) + b"".join(rs)

    out = {"dup_last_adapter": with_recs(recs + [recs[-1]]),
           "missing_last_adapter": with_recs(recs[:-1]),
           "no_adapters": with_recs([])}
    if len(recs) > 1:
        out["swapped_adapters"] = with_recs([recs[1], recs[0]] + recs[2:])
        out["dup_first_for_second"] = with_recs([recs[0], recs[0]] + recs[2:])
    b = bytearray(buf)
    b[ads[0][3]:ads[0][3] + 4] = struct.pack("<f", 0.0)
    out["alpha_zero"] = bytes(b)
    b = bytearray(buf)
    b[ads[-1][3]:ads[-1][3] + 4] = struct.pack("<f", -2.0)
    out["alpha_negative"] = bytes(b)
    assert tail == b"".join(recs)
    return out


def checkpoint_cases():
    import ctypes as C
    import json
    L = Ref.get()
    L.ref_make_checkpoint.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64, C.c_uint64]
    L.ref_checkpoint_probe.argtypes = [C.c_char_p] + [C.POINTER(C.c_uint64)] * 2 + [
        C.POINTER(C.c_int), C.POINTER(C.c_uint64)]

    def probe(path):
        fh, zh, k, o = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_uint64()
        rc = L.ref_checkpoint_probe(path.encode(), fh, zh, k, o)
        return {"status": rc, "file_hash": fh.value if rc == 0 else None,
                "frozen_hash": zh.value if rc == 0 else None, "format_kind": k.value,
                "offset": o.value if rc else None}

    expect = {}
    tmp = os.path.join(HERE, "_tmp.mlra")
    for name, task, bits, seed, group in CKPTS:
        path = os.path.join(HERE, name)
        rc = L.ref_make_checkpoint(path.encode(), task.encode(), bits, seed, group)
        assert rc == 0, L.ref_last_error()
        expect[name] = probe(path)
        buf = open(path, "rb").read()
        for cname, data in corruptions(buf).items():
            with open(tmp, "wb") as fh:
                fh.write(data)
            expect[f"{name}:{cname}"] = probe(tmp)
        for cname, data in structural_corruptions(buf).items():
            with open(tmp, "wb") as fh:
                fh.write(data)
            expect[f"{name}:{cname}"] = probe(tmp)
    os.remove(tmp)
    with open(os.path.join(HERE, "checkpoints.json"), "w") as fh:
        json.dump(expect, fh, indent=1, sort_keys=True)
    # the reference's pinned digests (acceptance.cpp:462-463, test_checkpoint.cpp:31-32)
    assert expect["golden.mlra"]["file_hash"] == 0xb48207d130703ee4
    assert expect["golden.mlra"]["frozen_hash"] == 0xa3d66a9e729158ff


def model_cases():
    """The parity transformer (model.cpp:226-292) pinned by the reference: the
    reference-made parity_b4.mlra with seeded non-zero adapters (so every dA /
    dB is live), then the reference's own model_loss + tape backward on seeded
    sequences -> loss and the flat trainable-parameter gradients."""
    import json
    from paper_2309_16119_b200.checkpoint import Checkpoint
    ck = Checkpoint.load(os.path.join(HERE, "parity_b4.mlra"))
    rng = np.random.default_rng(2309)
    n_grads = 0
    for i in range(len(ck)):
        r = ck.layer(i)
        ck.set_adapter(i, rng.normal(0.0, 0.15, (r.rows, r.rank)), rng.normal(0.0, 0.15, (r.cols, r.rank)))
        n_grads += r.rank * (r.rows + r.cols)
    path = os.path.join(HERE, "parity_b4_adapted.mlra")
    ck.save(path)
    cfg = json.loads(ck.config_json())
    dims = cfg.get("task_dims", {})
    seq, d = int(dims.get("seq_len", 8)), int(dims.get("d_model", 16))
    n = 6
    xs = rng.normal(0.0, 1.0, (n, seq, d))
    labels = rng.integers(0, 2, n).astype(np.int32)
    loss, grads = Ref.parity_loss_grads(path, xs, labels, n_grads)
    return dict(xs=xs, labels=labels, loss=np.array([loss]), grads=grads)


OPTQ_CASES = [  # rows, cols, m, bits, group, damping
    (6, 16, 24, 4, 8, 0.01), (33, 64, 100, 3, 32, 0.01), (64, 160, 300, 2, 0, 0.05),
    (40, 256, 512, 4, 128, 0.01), (16, 96, 64, 3, 32, 0.01), (10, 48, 200, 8, 16, 0.0),
    (7, 9, 12, 3, 3, 0.01)]


def optq_inputs(ci: int):
    """Seeded inputs of OPTQ case ci (regenerated by the tests; the fixture
    stores their digest, not the arrays)."""
    rows, cols, m, _, _, _ = OPTQ_CASES[ci]
    rng = np.random.default_rng(4242 + ci)
    w = rng.normal(0.0, 0.02, (rows, cols))
    x = rng.normal(0.0, 1.0, (m, cols))
    x[1:] = 0.6 * x[:-1] + 0.8 * x[1:]  # correlated calibration rows
    return w, x


def input_digest(*arrays) -> int:
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, np.float64).tobytes())
    return int.from_bytes(h.digest()[:8], "little")


def optq_cases():
    """quantize_optq / build_optq_workspace (quantize.cpp:186-255) by the reference."""
    out = {}
    for ci, (rows, cols, m, bits, group, damp) in enumerate(OPTQ_CASES):
        w, x = optq_inputs(ci)
        out[f"c{ci}_digest"] = np.array([input_digest(w, x)], np.uint64)
        words, scales, zeros = Ref.quantize_optq(w, x, bits, group, damp)
        if cols <= 100:  # the workspace itself, for the small cases (fixture size)
            h, u = Ref.optq_workspace(x, damp)
            out.update({f"c{ci}_h": h, f"c{ci}_u": u})
        out.update({f"c{ci}_words": words, f"c{ci}_scales": scales,
                    f"c{ci}_zeros": zeros,
                    f"c{ci}_meta": np.array([rows, cols, m, bits, group], np.int64),
                    f"c{ci}_damping": np.array([damp])})
    return out


def main():
    if not Ref.available():
        raise SystemExit("oracle/_ref/libmlra_ref.so missing: run `make -C oracle` with /root/reference present")
    if sys.argv[1:] == ["optq"]:
        np.savez_compressed(os.path.join(HERE, "optq.npz"), **optq_cases())
        return
    if sys.argv[1:] == ["checkpoints"]:
        checkpoint_cases()
        return
    if sys.argv[1:] == ["model"]:
        np.savez_compressed(os.path.join(HERE, "parity_model.npz"), **model_cases())
        return
    np.savez_compressed(os.path.join(HERE, "bitpack.npz"), **bitpack_cases())
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), **quant_cases())
    np.savez_compressed(os.path.join(HERE, "layer.npz"), **layer_cases())
    meta = {"mix_seed_11_ada9": Ref.get().ref_mix_seed(11, 0xADA9)}
    np.savez_compressed(os.path.join(HERE, "rng.npz"),
                        gaussian_seed7=Ref.gaussian(7, 3, 5),
                        gaussian_seed8_scaled=Ref.gaussian(8, 4, 4, 0.5, 0.02),
                        mix_seed_11_ada9=np.array([meta["mix_seed_11_ada9"]], np.uint64))
    checkpoint_cases()
    np.savez_compressed(os.path.join(HERE, "parity_model.npz"), **model_cases())
    np.savez_compressed(os.path.join(HERE, "optq.npz"), **optq_cases())
    for f in sorted(os.listdir(HERE)):
        if f.endswith((".npz", ".mlra", ".json")):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
