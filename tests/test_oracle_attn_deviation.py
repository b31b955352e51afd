"""Attention deviation (Fig. `ca_reduction` P:187-199; reading R16): the oracle's
Delta_attn(A_i, A_i^full) per layer, pinned by what the paper and the definitions fix:
- r = 100 % is full prefill, so every layer's deviation is exactly 0;
- layer 0's K/V and queries do not depend on cross-chunk attention: its deviation is the storage
  rounding of the chunk caches only;
- the deviation shrinks as the recompute ratio grows, and recomputing the HKVD tokens reduces it far more than
  recomputing the same number of random tokens (Insight 1) -- the shape of Fig. ca_reduction;
- attention_probs rows are distributions over the visible keys (brute-force softmax on one row)."""
import math

import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from synth import workload as W
from tests.helpers import oracle_model, request_inputs, shape

RATIOS = (0.0, 0.1, 0.2, 0.3, 0.5, 1.0)


def _case(seed):
    s = shape("tiny", n_layers=4)
    m = oracle_model(s, seed, "f32")
    req = W.Request([32, 32, 32], 16, seed, 0.15)
    tok, pos, cs, Kc, Vc = request_inputs(s, req, m, "f32")
    return s, m, req, tok, pos, cs, Kc, Vc


def test_attention_probs_is_the_masked_softmax():
    rng = np.random.default_rng(0)
    q, k = rng.normal(size=(3, 4, 8)), rng.normal(size=(10, 2, 8))
    qp, kp = np.array([2, 5, 9]), np.arange(10)
    A = O.attention_probs(q, qp, k, kp)
    for h in range(4):
        for r in range(3):
            vis = kp <= qp[r]
            logits = np.array([q[r, h] @ k[j, h // 2] / math.sqrt(8) for j in range(10)])
            e = np.where(vis, np.exp(logits - logits[vis].max()), 0.0)
            np.testing.assert_allclose(A[h, r], e / e.sum(), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_attention_deviation_curve(seed):
    s, m, req, tok, pos, cs, Kc, Vc = _case(seed)
    N, L = req.n_ctx, s.n_layers
    hkvd, rnd = [], []
    for r in RATIOS:
        ks = O.schedule(r, N, L)
        d = O.attention_deviation(m, tok, pos, cs, req.n_suffix, Kc, Vc, ks)
        dr = O.attention_deviation(m, tok, pos, cs, req.n_suffix, Kc, Vc, ks,
                                   force_sel=W.nested_selection(seed + 100, N, ks))
        assert d[0] < 1e-6 and dr[0] < 1e-6  # layer 0: only the fp32 storage of the chunk caches
        hkvd.append(d[1:].mean())
        rnd.append(dr[1:].mean())
    print(seed, "HKVD", np.round(hkvd, 5), "random", np.round(rnd, 5))
    assert hkvd[-1] < 1e-6 and rnd[-1] < 1e-6  # r = 100 %: full prefill (up to the fp32 storage of the caches)
    assert hkvd[0] == pytest.approx(rnd[0])       # r = 0: nothing recomputed, selection irrelevant
    assert all(a > b for a, b in zip(hkvd, hkvd[1:]))  # monotone in r
    for a, b in zip(hkvd[1:-1], rnd[1:-1]):       # HKVD beats random at every intermediate ratio
        assert a < 0.85 * b
