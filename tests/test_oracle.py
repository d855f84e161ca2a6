"""Pins the CPU oracle (oracle/vinf_oracle.c) before trusting it:
(1) the golden vectors frozen in the reference's own tests, and
(2) the reference library itself, compiled from its sources (oracle/_ref), bitwise.
Also checks the committed golden fixtures (tests/golden/) that travel to the GPU box."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_rng_goldens(oracle):
    # test_tensor.cpp:57-61
    assert oracle.fill_seeded(1, 0)[0] == np.float32(0.7666215896606445)
    assert oracle.fill_seeded(1, 1)[0] == np.float32(0.13312304019927979)
    t = oracle.tensor_from_seed((4, 2, 2, 3), 7)
    assert abs(float(np.sum(t.astype(np.float64))) - (-0.055846452713012695)) <= 1e-15


def test_rng_independent_restatement(oracle):
    # test_tensor.cpp:18-32 RefRng: double(top24) / 2^24 * 2 - 1
    M = (1 << 64) - 1
    s = 7
    want = []
    for _ in range(48):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        want.append(np.float32(2.0 * ((z >> 40) / float(1 << 24)) - 1.0))
    assert np.array_equal(oracle.fill_seeded(48, 7), np.array(want, np.float32))


def test_stream_offset(oracle):
    full = oracle.fill_seeded(96, 123)
    for start in (0, 1, 3, 6):
        assert np.array_equal(oracle.fill_seeded(96 - start * 12, 123, start * 12), full[start * 12:])


def test_token_set_goldens(oracle):
    # test_ops.cpp:302-354
    assert oracle.build_local_window(16, 64, 16) == list(range(8, 25))
    assert oracle.build_local_window(0, 64, 16) == list(range(0, 9))
    assert oracle.build_local_window(63, 64, 16) == list(range(55, 64))
    assert oracle.build_local_window(0, 1, 16) == [0]
    with pytest.raises(IndexError):
        oracle.build_local_window(5, 5, 16)
    assert oracle.build_global_index_set(24, 16) == [0, 1, 3, 4, 6, 7, 9, 10, 12, 13, 15, 16,
                                                     18, 19, 21, 22]
    assert oracle.build_global_index_set(32, 16) == [2 * j for j in range(16)]
    assert oracle.build_global_index_set(16, 16) == list(range(16))
    assert oracle.build_global_index_set(8, 0) == []
    with pytest.raises(ValueError):
        oracle.build_global_index_set(8, 9)
    # F=2300 and F=2304 sets differ
    assert oracle.build_global_index_set(2300, 16)[:6] == [0, 143, 287, 431, 575, 718]
    assert oracle.build_global_index_set(2304, 16)[:3] == [0, 144, 288]


def test_membership_goldens(oracle):
    # test_clip_parallel.cpp:66-81 style: members of the F=16, n=8 set in each quarter
    got = [oracle.global_members_in_range(16, 8, s, 4) for s in (0, 4, 8, 12)]
    assert got == [[0, 2], [0, 2], [0, 2], [0, 2]]
    assert oracle.global_members_in_range(48, 16, 24, 24) == [0, 3, 6, 9, 12, 15, 18, 21]


def test_oracle_bitwise_vs_reference(oracle, reference):
    C = 16
    x = oracle.tensor_from_seed((12, 2, 3, C), 3)
    assert np.array_equal(oracle.fill_seeded(1000, 5, 17), reference.fill_seeded(1000, 5, 17))
    bo, br = oracle.build_block(C, 3, 1), reference.build_block(C, 3, 4, 1)
    assert all(np.array_equal(a, b) for a, b in zip(bo.arrays(), br.arrays()))
    assert np.array_equal(oracle.temporal_conv(x, 3, bo.conv_w, bo.conv_b),
                          reference.conv_over_extended(x, 0, 12, 3, bo.conv_w, bo.conv_b))
    assert np.array_equal(oracle.conv_over_extended(x, 2, 7, 3, bo.conv_w, bo.conv_b),
                          reference.conv_over_extended(x, 2, 7, 3, bo.conv_w, bo.conv_b))
    assert np.array_equal(oracle.group_norm(x, 4, bo.gamma, bo.beta),
                          reference.group_norm(x, 4, bo.gamma, bo.beta))
    sc = float(np.float32(1) / np.sqrt(np.float32(C)))
    for t in (700.0, 800.0, 900.0):
        a, ca = oracle.dual_scope(x, t, bo.wq, bo.wk, bo.wv, bo.wo, sc, 6, 5, 4.0, 800.0, counters=True)
        b, cb = reference.dual_scope(x, t, bo.wq, bo.wk, bo.wv, bo.wo, sc, 6, 5, 4.0, 800.0, counters=True)
        assert np.array_equal(a, b) and ca == cb
    a, ra = oracle.attention_full(x, bo.wq, bo.wk, bo.wv, bo.wo, sc, True)
    b, rb = reference.attention_full(x, bo.wq, bo.wk, bo.wv, bo.wo, sc, True)
    assert np.array_equal(a, b) and np.array_equal(ra, rb)


def test_oracle_block_and_parallel_vs_reference(oracle, reference):
    C = 16
    x = oracle.tensor_from_seed((16, 2, 2, C), 9)
    bo = oracle.build_block(C, 3, 1)
    ya = oracle.block_forward(x, bo, 900.0, 4, n_local=4, n_global=4)
    yb = reference.block_forward(x, 3, 4, 1, 900.0, n_local=4, n_global=4)
    assert np.array_equal(ya, yb)
    yc = reference.block_forward(x, 3, 4, 1, 900.0, n_local=4, n_global=4, workers=4)
    assert np.abs(yc - yb).max() <= 1e-6  # GN stats combine differently across clips
    # the oracle's distributed attention form equals the reference's on worker 1
    sc = float(np.float32(1) / np.sqrt(np.float32(C)))
    g = oracle.build_global_index_set(16, 4)
    full = oracle.dual_scope(x, 900.0, bo.wq, bo.wk, bo.wv, bo.wo, sc, 4, 4, 10.0, 800.0)
    w1 = oracle.attention_parallel(16, 4, 1, x[4:8], x[2:4], x[8:10], x[g], 900.0, bo.wq, bo.wk,
                                   bo.wv, bo.wo, sc, 4, 4, 10.0, 800.0)
    assert np.array_equal(w1, full[4:8])


def test_traffic_closed_forms_vs_reference(oracle, reference):
    for (F, n, h, g) in [(16, 4, 2, 4), (48, 2, 8, 16), (192, 8, 8, 16), (64, 8, 1, 0)]:
        for w in range(n):
            assert oracle.predict_sync_traffic(F, n, h, g, w, 4096) == \
                reference.predict_sync_traffic(F, n, h, g, w, 4096)
            assert oracle.predict_groupnorm_traffic(F, n, 32, w) == \
                reference.predict_groupnorm_traffic(F, n, 32, w)
    # measured transport bytes of the reference's distributed block equal the closed form
    C, F, n = 16, 16, 4
    x = oracle.tensor_from_seed((F, 2, 2, C), 9)
    _, traffic = reference.block_forward(x, 3, 4, 1, 900.0, n_local=4, n_global=4, workers=n,
                                         traffic=True)
    fb = 2 * 2 * C * 4
    for w in range(n):
        conv = oracle.predict_sync_traffic(F, n, 1, 0, w, fb)[0]
        gn = oracle.predict_groupnorm_traffic(F, n, 4, w)[0]
        attn = oracle.predict_sync_traffic(F, n, 2, 4, w, fb)[0]
        assert traffic[w] == [conv, gn, attn]


def test_golden_fixtures_match_oracle(oracle):
    path = os.path.join(GOLDEN, "block_small.npz")
    if not os.path.exists(path):
        pytest.skip("fixtures not generated")
    z = np.load(path)
    C = int(z["C"])
    bo = oracle.build_block(C, 3, int(z["weight_seed"]))
    for key in ("stub_a", "conv_w", "wq", "wo"):
        assert np.array_equal(getattr(bo, key), z[key])
    y = oracle.block_forward(z["x"], bo, float(z["t"]), int(z["groups"]), n_local=int(z["n_local"]),
                             n_global=int(z["n_global"]))
    assert np.array_equal(y, z["y"])


@pytest.mark.parametrize("C,H,W", [(40, 3, 5), (12, 1, 7), (3, 2, 3)])
def test_oracle_vectorised_threaded_bitwise(oracle, reference, C, H, W, monkeypatch):
    # the checker vectorises across outputs and splits positions over threads
    # (vinf_oracle.c orc_rows / orc_parallel); every output must stay bitwise equal to the
    # reference's scalar loops, for ragged position blocks and C % 8 tails
    x = oracle.tensor_from_seed((10, H, W, C), 11)
    bo = oracle.build_block(C, 3, 2)
    groups = 1 if C % 4 else 4
    for threads in ("1", "3"):
        monkeypatch.setenv("ORC_THREADS", threads)
        assert np.array_equal(oracle.temporal_conv(x, 3, bo.conv_w, bo.conv_b),
                              reference.conv_over_extended(x, 0, 10, 3, bo.conv_w, bo.conv_b))
        sc = float(np.float32(1) / np.sqrt(np.float32(C)))
        a = oracle.dual_scope(x, 900.0, bo.wq, bo.wk, bo.wv, bo.wo, sc, 4, 3, 10.0, 800.0)
        b = reference.dual_scope(x, 900.0, bo.wq, bo.wk, bo.wv, bo.wo, sc, 4, 3, 10.0, 800.0)
        assert np.array_equal(a, b)
        assert np.array_equal(oracle.group_norm(x, groups, bo.gamma, bo.beta),
                              reference.group_norm(x, groups, bo.gamma, bo.beta))
