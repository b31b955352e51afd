"""Pins for the oracle's RoPE / realign (Appendix, footnote P:208-211)."""
import json
import os

import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from tests.conftest import GOLDEN


def test_rope_hand_values():
    """Hand-written cos/sin values (golden fixture) pin pairing, sign and the theta exponent (R8)."""
    with open(os.path.join(GOLDEN, "rope_hand_values.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        x = np.array(c["x"], dtype=np.float64)
        out = O.rope_rotate(x[None, :], np.array([c["m"]]), c["base"])[0]
        np.testing.assert_allclose(out, c["expect"], atol=1e-15, err_msg=str(c))


def test_rope_identity_and_norm():
    rng = np.random.default_rng(0)
    for d in (2, 8, 64, 128):
        x = rng.standard_normal((5, d))
        np.testing.assert_array_equal(O.rope_rotate(x, np.zeros(5), 10000.0), x)
        for m in (1, 7, 100, 9999):
            y = O.rope_rotate(x, np.full(5, m), 10000.0)
            np.testing.assert_allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-14)


def test_rope_relative_position_invariance():
    """Proposition P:2547-2561 / S:613: R(m+l)q . R(m)k = R(l)q . k, 1000 random samples."""
    rng = np.random.default_rng(1)
    for n in range(1000):
        d = (2, 8, 64)[n % 3]
        q, k = rng.standard_normal(d), rng.standard_normal(d)
        m = (0, 1, 17, 1000)[n % 4]
        l = int(rng.integers(0, 4096))
        lhs = O.rope_rotate(q[None], np.array([m + l]), 10000.0)[0] @ O.rope_rotate(k[None], np.array([m]), 10000.0)[0]
        rhs = O.rope_rotate(q[None], np.array([l]), 10000.0)[0] @ k
        assert abs(lhs - rhs) <= 1e-9 * (1 + abs(rhs))


def test_rope_not_position_free_for_sign_flip():
    """A transposed block (sin sign flipped) would still be a rotation; the score must depend on the
    SIGNED gap: R(l)q.k != R(-l)q.k for generic q, k."""
    rng = np.random.default_rng(2)
    q, k = rng.standard_normal(8), rng.standard_normal(8)
    a = O.rope_rotate(q[None], np.array([5]), 10000.0)[0] @ k
    b = O.rope_rotate(q[None], np.array([-5]), 10000.0)[0] @ k
    assert abs(a - b) > 1e-3


def test_realign_closed_form():
    """R(g - l) R(l) k = R(g) k: realigning a chunk-locally encoded key equals encoding it at g."""
    rng = np.random.default_rng(3)
    T, H, d = 40, 3, 16
    k = rng.standard_normal((T, H, d))
    loc = rng.integers(0, 512, T)
    glob = loc + rng.integers(0, 9000, T)
    k_loc = O.rope_rotate(k, loc[:, None], 10000.0)
    k_glob = O.rope_rotate(k, glob[:, None], 10000.0)
    np.testing.assert_allclose(O.realign(k_loc, loc, glob, 10000.0), k_glob, atol=1e-11)
    # position-free storage (src_pos = 0, R11) is the same call
    np.testing.assert_allclose(O.realign(k, np.zeros(T), glob, 10000.0), k_glob, atol=1e-11)
    # identity realignment
    np.testing.assert_array_equal(O.realign(k_loc, loc, loc, 10000.0), k_loc)


def test_realign_preserves_within_chunk_scores():
    """a chunk precomputed at [0, L) and realigned to [D, D+L) keeps its q.k scores."""
    rng = np.random.default_rng(4)
    L, d, D = 20, 32, 3000
    q, k = rng.standard_normal((L, d)), rng.standard_normal((L, d))
    p0 = np.arange(L)
    s0 = O.rope_rotate(q, p0, 10000.0) @ O.rope_rotate(k, p0, 10000.0).T
    k_re = O.realign(O.rope_rotate(k, p0, 10000.0), p0, p0 + D, 10000.0)
    s1 = O.rope_rotate(q, p0 + D, 10000.0) @ k_re.T
    np.testing.assert_allclose(s1, s0, atol=1e-9)


# ---- half-split RoPE (R9 variant; N3 loader conversion) ------------------------------------------------------
def test_rope_half_hand_values_and_invariants():
    # hd = 4, position 1: the pair (x0, x2) turns by theta_0 = 1 rad, (x1, x3) by theta_1 = base^(-1/2)
    y = O.rope_rotate_half(np.array([1.0, 0.0, 0.0, 0.0]), np.array(1.0), 10000.0)
    np.testing.assert_allclose(y, [np.cos(1.0), 0.0, np.sin(1.0), 0.0], atol=1e-15)
    y = O.rope_rotate_half(np.array([0.0, 1.0, 0.0, 0.0]), np.array(2.0), 10000.0)
    np.testing.assert_allclose(y, [0.0, np.cos(0.02), 0.0, np.sin(0.02)], atol=1e-15)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 8))
    # hd = 2: one pair, both conventions are the same rotation
    np.testing.assert_allclose(O.rope_rotate_half(x[:, :2], np.arange(50), 1e4), O.rope_rotate(x[:, :2], np.arange(50), 1e4))
    # norm preserved; q.k depends only on the position difference
    yq = O.rope_rotate_half(x, np.arange(50), 1e4)
    np.testing.assert_allclose(np.linalg.norm(yq, axis=1), np.linalg.norm(x, axis=1), rtol=1e-13)
    q, k = rng.standard_normal(8), rng.standard_normal(8)
    d1 = O.rope_rotate_half(q, np.array(17.0), 1e4) @ O.rope_rotate_half(k, np.array(5.0), 1e4)
    d2 = O.rope_rotate_half(q, np.array(112.0), 1e4) @ O.rope_rotate_half(k, np.array(100.0), 1e4)
    assert abs(d1 - d2) < 1e-12


def test_half_split_conversion_identity():
    """Loader conversion (paper_2405_16444_b200.dist): interleaved RoPE of the permuted projection equals the
    permuted half-split RoPE, and the inverse cache permutation restores the half-split order."""
    from paper_2405_16444_b200 import dist as D
    from synth import workload as W
    rng = np.random.default_rng(4)
    s = W.MODELS["tiny"]
    w = rng.standard_normal((s.qd + 2 * s.kvd, s.d_model))
    x = rng.standard_normal((9, s.d_model))
    pos = np.arange(9) + 30
    wp = D.interleave_rope_weights(w, s)
    z, zp = x @ w.T, x @ wp.T
    np.testing.assert_array_equal(zp[:, s.qd + s.kvd:], z[:, s.qd + s.kvd:])        # v rows untouched
    for h in range(s.n_q_heads + s.n_kv_heads):
        sl = slice(h * s.head_dim, (h + 1) * s.head_dim)
        half = O.rope_rotate_half(z[:, sl], pos, s.rope_theta)
        inter = O.rope_rotate(zp[:, sl], pos, s.rope_theta)
        np.testing.assert_allclose(D.interleave_rope_cache(inter, inverse=True), half, atol=1e-12)
    k = rng.standard_normal((3, 5, s.head_dim))
    np.testing.assert_array_equal(D.interleave_rope_cache(D.interleave_rope_cache(k), inverse=True), k)
