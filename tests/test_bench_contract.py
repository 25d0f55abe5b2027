"""The driver contract of bench.py's reference arm, runnable on CPU: one JSON
line with the reference's metric/config and the fields the driver reads."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not orc.Ref.available(), reason="reference library not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "tokens/s"
    assert line["warmup"] >= 3  # the contract's minimum
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"].startswith("cfg2")


def test_reference_arm_never_loads_the_product():
    """the reference arm must not map libmlra.so (the bench's word
    counts and synthetic codes are numpy only)."""
    code = ("import sys, bench, types; "
            "a = types.SimpleNamespace(workload='cfg2', bits=0, steps=1, warmup=0, scaling='weak'); "
            "import oracle.oracle as o; "
            "bench.cpu_reference_sample = lambda w, m, t, seed=1: (1.0, 'reference', 1); "
            "bench.run_reference(a, 0, 1); "
            "assert 'paper_2309_16119_b200' not in sys.modules; "
            "maps = open('/proc/self/maps').read(); assert 'libmlra.so' not in maps; print('clean')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "clean"


def test_both_arms_share_the_config_dict():
    import types
    sys.path.insert(0, ROOT)
    import bench
    for wl in bench.WORKLOADS:
        for scaling in ("weak", "strong"):
            a = types.SimpleNamespace(workload=wl, bits=0, scaling=scaling)
            w = bench.workload(a)
            c = bench._config_dict(w, a, 4)
            assert c["workload"] == w["name"]
            if scaling == "strong":
                assert c["global_tokens"] == w["tokens"]
            else:
                assert c["global_tokens"] == 4 * w["tokens"]
    # strong scaling shards the global tokens with sizes differing by <= 1
    a = types.SimpleNamespace(workload="cfg3", bits=0, scaling="strong")
    w = bench.workload(a)
    ms = [bench.tokens_of(w, a, r, 3)[0] for r in range(3)]
    assert sum(ms) == 8192 and max(ms) - min(ms) <= 1


@pytest.mark.parametrize("rows,cols,bits", [(8, 4096, 3), (5, 11008, 3), (3, 8192, 4), (4, 512, 2),
                                            (2, 256, 8)])
def test_bench_parity_restatement_matches_oracle(rows, cols, bits):
    """bench.py's own numpy dequantizer (used for the per-run parity bit) is the
    oracle's dequantize bit for bit."""
    sys.path.insert(0, ROOT)
    import bench
    words, sc, z = bench.synthetic_codes(rows, cols, bits, 128, seed=rows + bits)
    want = orc.dequantize(words, rows, cols, bits, 128, sc, z)
    got = np.vstack([bench._deq_rows(words, cols, bits, 128, sc, z, r, r + 1) for r in range(rows)])
    assert np.array_equal(got, want)
    assert np.array_equal(bench._deq_rows(words, cols, bits, 128, sc, z, 0, rows), want)
    assert np.array_equal(bench._bf16(want), orc.bf16_round(want.astype(np.float32)))


def test_bench_parity_check_accepts_exact_and_rejects_wrong():
    sys.path.insert(0, ROOT)
    import bench
    w = dict(bench.WORKLOADS["cfg1"], layers=[("lin", 256, 512)], rank=8)
    rows, cols, m, r = 256, 512, 64, 8
    words, sc, z = bench.synthetic_codes(rows, cols, 4, 128, seed=3)
    rng = np.random.default_rng(0)
    x = bench._bf16(rng.standard_normal((m, cols)))
    dy = bench._bf16(rng.standard_normal((m, rows)))
    a = (0.02 * rng.standard_normal((rows, r))).astype(np.float32)
    b = (0.02 * rng.standard_normal((cols, r))).astype(np.float32)
    wex = bench._deq_rows(words, cols, 4, 128, sc, z, 0, rows)
    s = bench.ALPHA / r
    y = bench._bf16(x @ bench._bf16(wex).T + bench._bf16(s * x @ b) @ bench._bf16(a).T)
    dx = bench._bf16(dy @ bench._bf16(wex) + bench._bf16(s * dy @ a) @ bench._bf16(b).T)
    da = s * dy.T @ (x @ b)
    db = s * x.T @ (dy @ a)
    rec = [((words, sc, z, rows, cols), (x, y, dy, dx, a, b, da, db))]
    ok, worst, _ = bench.parity_check(rec, w)
    assert ok, worst
    rec = [((words, sc, z, rows, cols), (x, 1.01 * y, dy, dx, a, b, da, db))]
    assert not bench.parity_check(rec, w)[0]


@pytest.mark.skipif(not orc.Ref.available(), reason="reference library not built")
def test_reference_arm_self_launches_ranks():
    """--gpus 2 outside torchrun re-launches as 2 ranks; rank 0 alone prints."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "1", "--workload", "cfg1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"


@pytest.mark.gpu
def test_bench_gpus_2_runs_two_ranks():
    """`bench.py --gpus 2` launches two ranks itself and reports
    n_gpus 2 (on the 1-GPU box both ranks share cuda:0 over gloo); strong
    scaling splits cfg3's 8192 tokens."""
    env = dict(os.environ, MLRA_DIST_BACKEND="gloo", MLRA_NO_NUMA_BIND="1")
    for extra, tok in ((["--workload", "cfg1"], 512), (["--workload", "cfg3", "--scaling", "strong"], 4096)):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
                            "2", "--warmup", "3", "--no-cpu-baseline", "--no-parity"] + extra,
                           capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, r.stdout[-2000:]
        line = json.loads(lines[0])
        assert line["n_gpus"] == 2 and line["comm"] == {"backend": "gloo", "nranks": 2}
        assert line["arm"]["tokens_this_rank"] == tok and line["value"] > 0
        assert line["scaling"] == ("strong" if "strong" in extra else "weak")
