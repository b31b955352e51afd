"""Pins for the oracle's whole blend (§3.2, §3.3) against what the
paper and the mathematics fix: r = 100 % is full prefill, r = 0 is the realigned cache, a single
chunk is prefix reuse, sets nest, untouched entries are bitwise the realigned cache, and compute
is proportional to the recompute ratio."""
import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from synth import workload as W
from tests.helpers import oracle_model, request_inputs, shape


def _setup(name="tiny", seed=0, lens=(32, 32, 32), n_suf=0, dtype="f32", **over):
    s = shape(name, **over)
    m = oracle_model(s, seed, dtype)
    req = W.Request(list(lens), n_suf, seed, 0.15)
    tok, pos, cs, Kc, Vc = request_inputs(s, req, m, dtype)
    return s, m, req, tok, pos, cs, Kc, Vc


@pytest.mark.parametrize("seed", range(20))
def test_full_ratio_equals_full_prefill(seed):
    """S:290 / S:611: r = 1 -> KV^new = KV^full and h = full-prefill h (20 seeds, tiny config)."""
    s, m, req, tok, pos, cs, Kc, Vc = _setup(seed=seed)
    ks = O.schedule(1.0, req.n_ctx, s.n_layers)
    # chunk caches in fp64 (no storage rounding) so the identity is exact up to fp64 rounding
    Kc64, Vc64 = O.precompute_chunk_caches(m, tok, cs)
    res = O.blend_forward(m, tok, pos, cs, 0, Kc64, Vc64, ks)
    Kf, Vf, hf = O.full_prefill(m, tok, pos)
    np.testing.assert_allclose(res.K, Kf, atol=1e-11)
    np.testing.assert_allclose(res.V, Vf, atol=1e-11)
    np.testing.assert_allclose(res.h_final, hf, atol=1e-10)


def test_full_ratio_with_suffix_and_gqa():
    s, m, req, tok, pos, cs, Kc, Vc = _setup(lens=(17, 40, 9), n_suf=5, n_kv_heads=2, n_layers=4)
    Kc64, Vc64 = O.precompute_chunk_caches(m, tok[:req.n_ctx], cs)
    res = O.blend_forward(m, tok, pos, cs, 5, Kc64, Vc64, O.schedule(1.0, req.n_ctx, 4))
    Kf, Vf, hf = O.full_prefill(m, tok, pos)
    np.testing.assert_allclose(res.K, Kf, atol=1e-11)
    np.testing.assert_allclose(res.h_final, hf, atol=1e-10)


def test_zero_ratio_is_realigned_cache():
    """r = 0: KV^new = concatenated chunk caches after realignment; V bitwise (BASELINE north_star)."""
    s, m, req, tok, pos, cs, Kc, Vc = _setup(seed=4)
    res = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, O.schedule(0.0, req.n_ctx, s.n_layers))
    loc = req.local_positions()
    for i in range(s.n_layers):
        np.testing.assert_array_equal(res.V[i], Vc[i])
        np.testing.assert_allclose(res.K[i], O.realign(Kc[i], loc, pos, s.rope_theta), atol=0)
        assert len(res.sel[i]) == (req.n_ctx if i == 0 else 0)


@pytest.mark.parametrize("r", [0.0, 0.15, 0.5])
def test_single_chunk_equals_prefix_reuse(r):
    """S:291 / S:612: one chunk (+ suffix) -> blend equals full prefill for any r (prefix caching)."""
    s, m, req, tok, pos, cs, _, _ = _setup(lens=(40,), n_suf=6, n_layers=3, seed=9)
    Kc64, Vc64 = O.precompute_chunk_caches(m, tok[:req.n_ctx], cs)
    res = O.blend_forward(m, tok, pos, cs, 6, Kc64, Vc64, O.schedule(r, req.n_ctx, 3))
    Kf, Vf, hf = O.full_prefill(m, tok, pos)
    np.testing.assert_allclose(res.K, Kf, atol=1e-11)
    np.testing.assert_allclose(res.V, Vf, atol=1e-11)
    np.testing.assert_allclose(res.h_final, hf[np.concatenate([res.sel[-1], 40 + np.arange(6)])], atol=1e-10)


def test_structural_invariants():
    """S_{i+1} subset of S_i, |S_i| = k_i; entries outside S_i are bitwise the realigned
    cache; first-chunk deviation is 0 (prefix stability, R7); layer-0 K/V equal the cache."""
    s, m, req, tok, pos, cs, Kc, Vc = _setup(seed=5, n_layers=5, lens=(24, 30, 18))
    ks = O.schedule(0.3, req.n_ctx, 5)
    res = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks)
    loc = req.local_positions()
    for i in range(1, 5):
        assert len(res.sel[i]) == ks[i]
        assert set(res.sel[i]) <= set(res.cand[i])
        np.testing.assert_array_equal(res.cand[i], res.sel[i - 1] if i > 1 else np.arange(req.n_ctx))
        untouched = np.setdiff1d(np.arange(req.n_ctx), res.sel[i])
        np.testing.assert_array_equal(res.V[i][untouched], Vc[i][untouched])
        np.testing.assert_array_equal(res.K[i][untouched],
                                      O.realign(Kc[i], loc, pos, s.rope_theta)[untouched])
    Kc64, Vc64 = O.precompute_chunk_caches(m, tok, cs)
    r64 = O.blend_forward(m, tok, pos, cs, 0, Kc64, Vc64, ks)
    first = r64.cand[1] < cs[1]
    assert np.abs(r64.dev[1][first]).max() < 1e-20
    assert r64.dev[1][~first].max() > 1e-6
    # layer 0 fresh K/V of context rows equal the realigned cache (deviation identically 0)
    _, k0, v0 = O.qkv(m, 0, m.embed[tok], pos)
    np.testing.assert_allclose(O.kv_deviation(k0, v0, r64.K[0], r64.V[0]), 0, atol=1e-20)


def test_hkvd_are_top_deviation_tokens():
    """S_i is exactly the top-k_i of Delta_kv over C_i (brute-force re-rank) at every layer."""
    s, m, req, tok, pos, cs, Kc, Vc = _setup(seed=6, n_layers=4)
    ks = O.schedule(0.25, req.n_ctx, 4)
    res = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks)
    for i in range(1, 4):
        order = sorted(range(len(res.cand[i])), key=lambda j: (-res.dev[i][j], res.cand[i][j]))
        assert sorted(res.cand[i][order[:ks[i]]].tolist()) == res.sel[i].tolist()


def test_replay_mode_uses_forced_selection():
    s, m, req, tok, pos, cs, Kc, Vc = _setup(seed=7, n_layers=3)
    ks = O.schedule(0.2, req.n_ctx, 3)
    free = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks)
    forced = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks, force_sel=free.sel)
    np.testing.assert_array_equal(forced.K, free.K)
    np.testing.assert_array_equal(forced.h_final, free.h_final)
    other = [None, np.arange(ks[1]), np.arange(ks[2])]
    alt = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks, force_sel=other)
    assert alt.sel[1].tolist() == list(range(ks[1]))
    with pytest.raises(ValueError):
        O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks, force_sel=[None, np.arange(ks[1]), np.array([90, 95])])


@pytest.mark.parametrize("r", [0.10, 0.15, 0.20])
def test_mac_proportionality(r):
    """S:316 / P:159-161: blend MACs / full-prefill MACs in [r - 0.05, r + 0.10] (32-layer model)."""
    s = shape("tiny", n_layers=32, d_model=32, n_q_heads=4, n_kv_heads=2, head_dim=8, d_ff=64)
    m = oracle_model(s, 1)
    req = W.Request([40, 40, 40], 0, 1, r)
    tok, pos, cs = req.tokens(s.vocab), req.global_positions(), req.chunk_starts()
    Kc = np.zeros((32, 120, 2, 8))
    res = O.blend_forward(m, tok, pos, cs, 0, Kc, Kc, O.schedule(r, 120, 32), count_macs=True)
    ratio = res.macs / O.full_prefill_macs(m, tok, pos)
    assert r - 0.05 <= ratio <= r + 0.10, ratio


@pytest.mark.parametrize("name,lens,layers,ratio,threads", [("tiny", (32, 32, 32), 3, 0.15, 1),
                                                           ("tiny", (20, 45, 31), 4, 0.5, 4),
                                                           ("small", (100, 77, 60), 3, 0.3, 8)])
def test_replay_rows_equals_forced_blend(name, lens, layers, ratio, threads):
    """blend_replay_rows (the row-restricted replay used at full model width) equals blend_forward with the
    same forced selections on every row it returns: KV^new of every layer, Delta_kv of every evaluated
    candidate, and the final h rows (a subset of S_{L-1} on the last layer)."""
    s = shape(name, n_layers=layers)
    m = oracle_model(s, 3, "f32")
    req = W.Request(list(lens), 0, 3, ratio)
    tok, pos, cs, Kc, Vc = request_inputs(s, req, m, "f32")
    N = req.n_ctx
    ks = O.schedule(ratio, N, layers)
    S = W.nested_selection(3, N, ks)
    d1 = W.sample_rows(3, 0x77, N, 11)
    full = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks, force_sel=S)
    last = S[-1][::3]
    rr = O.blend_replay_rows(tok, pos, cs, Kc, Vc, S, lambda i: m, m.embed[tok], dev_rows_1=d1,
                             h_rows_last=last, threads=threads)
    np.testing.assert_allclose(rr["K"], full.K, rtol=0, atol=1e-12)
    np.testing.assert_allclose(rr["V"], full.V, rtol=0, atol=1e-12)
    for i in range(1, layers):
        untouched = np.setdiff1d(np.arange(N), S[i])
        np.testing.assert_array_equal(rr["V"][i][untouched], Vc[i][untouched])
        rows, dv = rr["dev"][i]
        pos_in = np.searchsorted(full.cand[i], rows)
        np.testing.assert_allclose(dv, full.dev[i][pos_in], rtol=1e-12, atol=1e-12)
        assert set(full.sel[i]) == set(S[i].tolist())
    assert set(d1.tolist()) <= set(rr["dev"][1][0].tolist())
    h0 = O.blend_replay_rows(tok, pos, cs, Kc[:1], Vc[:1], S[:1], lambda i: m, m.embed[tok])["h"]
    r2 = O.blend_replay_rows(tok, pos, cs, Kc, Vc, S, lambda i: m, None, dev_rows_1=d1, h_rows_last=last, h0=h0)
    np.testing.assert_allclose(r2["h"], rr["h"], rtol=1e-11, atol=1e-11)
    np.testing.assert_array_equal(rr["h_rows"], last)
    np.testing.assert_allclose(rr["h"], full.h_final[np.searchsorted(S[-1], last)], rtol=1e-11, atol=1e-11)


def test_nested_selection_recipe():
    """The forced-selection recipe nests and has the scheduled sizes (an input generator, no method)."""
    ks = O.schedule(0.3, 500, 6)
    S = W.nested_selection(1, 500, ks)
    assert len(S) == 6 and np.array_equal(S[0], np.arange(500))
    for i in range(1, 6):
        assert len(S[i]) == ks[i] and np.all(np.diff(S[i]) > 0) and set(S[i]) <= set(S[i - 1])
