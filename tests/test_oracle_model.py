"""Pins for the oracle's transformer pieces and full prefill (§2 Background P:292-316).

The independent reference here is torch's own library routines in fp64 on CPU
(F.rms_norm, F.scaled_dot_product_attention, F.silu, complex-multiply RoPE via
torch.polar) — a different formulation of each step, so a dropped term, a wrong
index or a transposed operand in the oracle shows up as a mismatch."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import cacheblend_oracle as O
from synth import workload as W
from tests.helpers import oracle_model, shape


def torch_prefill(m: O.Model, tok, pos):
    """Textbook decoder forward written with torch library routines (fp64)."""
    d, hq, hk, hd = m.d_model, m.n_q_heads, m.n_kv_heads, m.head_dim
    T = len(tok)
    posT = torch.tensor(np.asarray(pos), dtype=torch.float64)
    inv = torch.tensor(m.rope_theta, dtype=torch.float64) ** (
        -torch.arange(0, hd, 2, dtype=torch.float64) / hd)
    rot = torch.polar(torch.ones(T, hd // 2, dtype=torch.float64), posT[:, None] * inv[None, :])

    def rope(x):  # x [T][H][hd], pairs (2i, 2i+1) as complex numbers
        xc = torch.view_as_complex(x.reshape(T, x.shape[1], hd // 2, 2).contiguous())
        return torch.view_as_real(xc * rot[:, None, :]).reshape(T, x.shape[1], hd)

    h = torch.tensor(m.embed[np.asarray(tok)])
    Ks, Vs = [], []
    for w in m.layers:
        w = {k: torch.tensor(v) for k, v in w.items()}
        x = F.rms_norm(h, (d,), w["attn_norm"], eps=m.rms_eps)
        q = rope((x @ w["wq"].T).reshape(T, hq, hd))
        k = rope((x @ w["wk"].T).reshape(T, hk, hd))
        v = (x @ w["wv"].T).reshape(T, hk, hd)
        a = F.scaled_dot_product_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1),
                                           is_causal=True, enable_gqa=True)
        h = h + a.transpose(0, 1).reshape(T, hq * hd) @ w["wo"].T
        x = F.rms_norm(h, (d,), w["mlp_norm"], eps=m.rms_eps)
        h = h + (F.silu(x @ w["wg"].T) * (x @ w["wu"].T)) @ w["wd"].T
        Ks.append(k.numpy())
        Vs.append(v.numpy())
    return np.stack(Ks), np.stack(Vs), h.numpy()


@pytest.mark.parametrize("name,over", [("tiny", {}), ("tiny", {"n_kv_heads": 2}),
                                       ("tiny", {"n_kv_heads": 1, "n_layers": 3})])
def test_full_prefill_matches_torch(name, over):
    s = shape(name, **over)
    m = oracle_model(s, seed=11, dtype="f32")
    tok = np.random.default_rng(0).integers(0, s.vocab, 37)
    pos = np.arange(37)
    K, V, h = O.full_prefill(m, tok, pos)
    K2, V2, h2 = torch_prefill(m, tok, pos)
    np.testing.assert_allclose(K, K2, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(V, V2, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(h, h2, rtol=1e-10, atol=1e-10)


def test_rms_norm_closed_form():
    g = np.linspace(0.5, 1.5, 8)
    for c in (2.0, -3.0, 1e-3):
        out = O.rms_norm(np.full((1, 8), c), g, 1e-5)[0]
        np.testing.assert_allclose(out, c / np.sqrt(c * c + 1e-5) * g, rtol=1e-14)


def test_attention_closed_forms():
    rng = np.random.default_rng(5)
    T, hq, hk, hd = 9, 4, 2, 8
    v = rng.standard_normal((T, hk, hd))
    q = rng.standard_normal((T, hq, hd))
    pos = np.arange(T)
    # identical keys -> uniform weights -> running mean of visible V rows
    k = np.tile(rng.standard_normal((1, hk, hd)), (T, 1, 1))
    out = O.causal_attention(q, pos, k, v, pos).reshape(T, hq, hd)
    for t in range(T):
        for h in range(hq):
            np.testing.assert_allclose(out[t, h], v[:t + 1, h // 2].mean(axis=0), atol=1e-12)
    # the first query sees only key 0 -> output = v[0] exactly
    k = rng.standard_normal((T, hk, hd))
    out = O.causal_attention(q[:1], pos[:1], k, v, pos).reshape(1, hq, hd)
    np.testing.assert_allclose(out[0, 0], v[0, 0], atol=1e-15)
    np.testing.assert_allclose(out[0, 3], v[0, 1], atol=1e-15)


def test_sparse_query_rows_equal_dense_rows():
    """Sparse-query attention (selected queries over all keys) = the same rows of dense causal
    attention computed by brute force (per-query loops, textbook softmax)."""
    rng = np.random.default_rng(6)
    T, hq, hk, hd = 23, 4, 1, 8
    q, k, v = rng.standard_normal((T, hq, hd)), rng.standard_normal((T, hk, hd)), rng.standard_normal((T, hk, hd))
    pos = np.arange(T) * 3 + 5
    sel = np.array([2, 7, 8, 19, 22])
    out = O.causal_attention(q[sel], pos[sel], k, v, pos).reshape(len(sel), hq, hd)
    for r, t in enumerate(sel):
        for h in range(hq):
            sc = [float(q[t, h] @ k[j, 0]) / np.sqrt(hd) for j in range(t + 1)]
            mx = max(sc)
            e = [np.exp(s - mx) for s in sc]
            ref = sum(e[j] * v[j, 0] for j in range(t + 1)) / sum(e)
            np.testing.assert_allclose(out[r, h], ref, atol=1e-12)


def test_causality_and_prefix_stability():
    """perturbing token t changes no K/V of tokens < t; prefill(prefix ++ suffix) restricted to
    the prefix equals prefill(prefix) (P:379 'KV cache of a prefix is not affected')."""
    s = shape("tiny")
    m = oracle_model(s, seed=3)
    tok = np.random.default_rng(1).integers(0, s.vocab, 30)
    K, V, _ = O.full_prefill(m, tok, np.arange(30))
    tok2 = tok.copy()
    tok2[17] = (tok2[17] + 1) % s.vocab
    K2, V2, _ = O.full_prefill(m, tok2, np.arange(30))
    np.testing.assert_allclose(K2[:, :17], K[:, :17], atol=1e-13)
    assert np.abs(K2[:, 17:] - K[:, 17:]).max() > 1e-6
    Kp, Vp, _ = O.full_prefill(m, tok[:12], np.arange(12))
    np.testing.assert_allclose(Kp, K[:, :12], atol=1e-13)
    np.testing.assert_allclose(Vp, V[:, :12], atol=1e-13)


def test_generator_recipe_statistics():
    """The synthetic weights follow the stated recipe (uniform/sqrt(fan_in), gains 1 +- 0.1)."""
    s = shape("tiny")
    w = W.layer_weights(s, 0, 7, "f32")
    assert abs(np.abs(w["wq"]).max() - 1 / np.sqrt(s.d_model)) < 1e-2
    assert 0.9 <= w["attn_norm"].min() and w["attn_norm"].max() < 1.1
