"""Test helpers: build oracle-side models/requests from the shared seeded generators."""
from __future__ import annotations

import dataclasses

import numpy as np

from oracle import cacheblend_oracle as O
from synth import workload as W


def shape(name: str, **over) -> W.ModelShape:
    s = W.MODELS[name]
    return dataclasses.replace(s, **over) if over else s


def oracle_model(s: W.ModelShape, seed: int, dtype: str = "f32") -> O.Model:
    layers = [W.layer_weights(s, i, seed, dtype) for i in range(s.n_layers)]
    return O.Model.build(s, W.embed_weights(s, seed, dtype), layers)


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp64 oracle outputs to the storage dtype (used only to build stored inputs)."""
    from synth import counter_rng as rng
    x32 = np.asarray(x, dtype=np.float32)
    if dtype == "f32":
        return x32
    return rng.bf16_bits_to_f32(rng.to_bf16_bits(x32)).reshape(x32.shape)


def request_inputs(s: W.ModelShape, req: W.Request, model: O.Model, dtype: str):
    """tok, pos, chunk_starts, and the stored chunk caches (oracle precompute, rounded to dtype)."""
    tok = req.tokens(s.vocab)
    pos = req.global_positions()
    cs = req.chunk_starts()
    Kc, Vc = O.precompute_chunk_caches(model, tok[:req.n_ctx], cs)
    return tok, pos, cs, round_to(Kc, dtype), round_to(Vc, dtype)


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def topk_tokens(dev, cand, k: int) -> np.ndarray:
    """Brute-force top-k (largest dev first, ties -> lower token), sorted ascending: the property the GPU's
    selection must satisfy on its OWN reported deviations (test-side code, not the oracle)."""
    dev = np.asarray(dev, np.float64)
    cand = np.asarray(cand)
    order = np.lexsort((cand, -dev))
    return np.sort(cand[order[:k]])


def band_check(gpu_sel, gpu_dev, ora_dev, cand, k: int):
    """Selection parity when the deviations carry bf16 error (R14): the GPU's S_i may differ from the oracle's
    top-k only on tokens whose oracle Delta_kv lies within the band E + |cut_gpu - cut_oracle| of the oracle's
    k-th value, E = the measured max |Delta_kv(gpu) - Delta_kv(oracle)| over the candidates. (A token the GPU
    keeps and the oracle drops has oracle Delta_kv in [cut_gpu - E, cut_oracle], and symmetrically.)
    Returns (ok, number of flips, band)."""
    gd = np.asarray(gpu_dev, np.float64)
    od = np.asarray(ora_dev, np.float64)
    cand = np.asarray(cand)
    osel = topk_tokens(od, cand, k)
    flips = np.setxor1d(np.asarray(gpu_sel), osel)
    if k == 0 or len(flips) == 0:
        return True, int(len(flips)), 0.0
    E = float(np.abs(gd - od).max())
    cut_o = np.sort(od)[::-1][k - 1]
    cut_g = np.sort(gd)[::-1][k - 1]
    band = E + abs(cut_g - cut_o)
    d_of = dict(zip(cand.tolist(), od.tolist()))
    ok = all(abs(d_of[t] - cut_o) <= band for t in flips.tolist())
    return ok, int(len(flips)), band
