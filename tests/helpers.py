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
