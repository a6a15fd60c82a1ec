"""Pins for oracle/rng.py and oracle/srht.py (readings G-6..G-10)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import rng, srht

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_vector():
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    out = rng.splitmix64_stream(g["seed"], 5)
    assert [str(x) for x in out] == g["outputs"]
    # the counter hash h(key, i) is output i of SplitMix64(state = key)
    assert [rng.h(g["seed"], i) for i in range(5)] == out


def test_signs_vectorized_equals_scalar_hash():
    k = rng.key(77, rng.TAG_SIGN)
    ref = np.array([-1 if rng.h(k, t) >> 63 else 1 for t in range(300)], dtype=np.int8)
    assert np.array_equal(rng.signs(77, 1024)[:300], ref)
    assert np.array_equal(rng.signs(77, 1024, start=100, count=50), ref[100:150])


def test_signs_balanced():
    N = 1 << 16
    d = rng.signs(5, N).astype(np.float64)
    assert abs(d.mean()) <= 4 / math.sqrt(N)


def test_rows_structure_and_floyd():
    for seed, N, s in [(1, 1024, 16), (3003, 1 << 24, 400), (9, 64, 64), (2, 8, 1)]:
        r = rng.rows(seed, N, s)
        assert len(r) == s and len(np.unique(r)) == s
        assert np.all(np.diff(r) > 0) and r[0] >= 0 and r[-1] < N
    assert np.array_equal(rng.rows(9, 64, 64), np.arange(64))   # s = N: everything
    with pytest.raises(ValueError):
        rng.rows(1, 8, 9)


def test_rows_floyd_hand_trace():
    """Floyd's sampler step by step on the published SplitMix64 stream (two
    collisions: the 'take j' branch runs at j = 2 and j = 3); a uniform but
    different sampler fails this."""
    g = json.load(open(os.path.join(GOLD, "floyd_trace.json")))
    qs = rng.splitmix64_stream(g["state"], g["s"])
    for st, q in zip(g["trace"], qs):
        assert f"{q / 2.0 ** 64:.4f}" == st["q_over_2_64"]
        assert (q * (st["j"] + 1)) >> 64 == st["t"]
    assert rng.rows_from_key(g["state"], g["N"], g["s"]).tolist() == g["rows"]
    assert sorted(st["taken"] for st in g["trace"]) == g["rows"]


def test_rows_uniform_chi2():
    # each index of [0, 32) should be chosen with probability s/N = 1/4
    N, s, T = 32, 8, 4000
    counts = np.zeros(N)
    for seed in range(T):
        counts[rng.rows(seed, N, s)] += 1
    expct = T * s / N
    chi2 = ((counts - expct) ** 2 / expct).sum()
    assert chi2 < 70    # 31 dof: p ~ 1e-4


def test_fwht_equals_dense_sylvester():
    rs = np.random.default_rng(0)
    for N in [1, 2, 4, 64, 1024, 4096]:
        x = rs.standard_normal(N)
        Hd = srht.hadamard_dense(N) if N <= 1024 else None
        y = srht.fwht(x)
        if Hd is not None:
            assert np.allclose(y, Hd @ x, rtol=0, atol=1e-12 * max(1, np.abs(x).sum()))
            assert np.array_equal(Hd @ Hd, N * np.eye(N))            # H^2 = N I
        assert np.allclose(srht.fwht(y), N * x, rtol=1e-12, atol=1e-12 * N)


def test_fwht_hand_case_spec_179():
    # n = 4, s = 4, signs +, x = e_1 -> first Hadamard column / sqrt(s)
    th = srht.SRHT(4, 4, seed=0)
    th.signs = np.ones(4, dtype=np.int8)
    y = th.apply(np.array([1.0, 0, 0, 0]))
    assert np.allclose(y, np.array([1, 1, 1, 1]) / 2.0)


def test_srht_isometry_at_s_equals_N_and_padding():
    rs = np.random.default_rng(1)
    for n in [8, 100, 1000]:
        N = srht.next_pow2(n)
        th = srht.SRHT(n, N, seed=n)
        for _ in range(5):
            x = rs.standard_normal(n)
            assert abs(np.linalg.norm(th.apply(x)) - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)


def test_srht_linear_and_zero():
    th = srht.SRHT(1000, 120, seed=4)
    x = np.random.default_rng(2).standard_normal(1000)
    assert np.array_equal(th.apply(2 * x), 2 * th.apply(x))
    assert np.array_equal(th.apply(np.zeros(1000)), np.zeros(120))


def test_srht_expected_norm_monte_carlo():
    x = np.random.default_rng(3).standard_normal(500)
    vals = [np.linalg.norm(srht.SRHT(500, 64, seed=s).apply(x)) ** 2 for s in range(300)]
    assert abs(np.mean(vals) / (x @ x) - 1) < 0.05


def test_srht_embedding_quality():
    # Subspace embedding: for an orthonormal n x m Q and
    # s = 2m, the singular values of Theta Q concentrate in the
    # Marchenko-Pastur interval [1 - sqrt(m/s), 1 + sqrt(m/s)] = [0.29, 1.71]
    # (cond ~ 5.8).  (SPEC S:185's "cond <= 3" is not attainable at s = 2m.)
    Q, _ = np.linalg.qr(np.random.default_rng(4).standard_normal((4096, 50)))
    good = 0
    for seed in range(40):
        sv = np.linalg.svd(srht.SRHT(4096, 100, seed).apply(Q), compute_uv=False)
        good += (sv[0] <= 1.9) and (sv[-1] >= 0.2)
    assert good >= 38


def test_row_entry_matches_full_transform():
    n = 3000
    th = srht.SRHT(n, 37, seed=11)
    x = np.random.default_rng(5).standard_normal(n)
    full = th.apply(x)
    for q in [0, 5, 36]:
        assert abs(th.row_entry(int(th.rows[q]), x) - full[q]) <= 1e-12 * np.abs(x).sum()


def test_pruned_tile_decomposition():
    """The identity the GPU kernels rely on: for aligned tiles
    of T consecutive indices, (H_N D x)_r = sum_tiles (-1)^popcount((r>>logT)
    & tile) * (H_T D x_tile)_(r mod T).  Checked against the full FWHT, with
    a non-multiple-of-T length (partial last tile zero-filled)."""
    n, T = 3000, 256
    th = srht.SRHT(n, 37, seed=13)
    x = np.random.default_rng(6).standard_normal(n)
    dx = np.zeros(th.N)
    dx[:n] = x * th.signs[:n]
    acc = np.zeros(37)
    for tile in range(th.N // T):
        out = srht.fwht(dx[tile * T:(tile + 1) * T])
        for q, r in enumerate(th.rows):
            par = bin((int(r) >> 8) & tile).count("1") & 1
            acc[q] += (-1.0 if par else 1.0) * out[int(r) % T]
    assert np.allclose(acc * th.scale, th.apply(x), rtol=1e-13, atol=1e-13)
