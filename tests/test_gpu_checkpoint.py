"""A Hugging Face checkpoint through the CUDA path: checkpoint.load onto the GPU, chunk caches
produced by the engine (transformers) and converted to the library's RoPE order, cb_blend_forward, then the
blended KV converted back and handed to the engine for a decode step. Checked against the fp64 oracle
on the loaded weights and against transformers' own full prefill."""
import types

import numpy as np
import pytest
import torch

from oracle import cacheblend_oracle as O
from paper_2405_16444_b200 import checkpoint as C
from tests import hf_model as H
from tests.gpu_helpers import run_blend
from tests.helpers import band_check, rel_err, round_to
from tests.test_checkpoint import engine_chunk_caches, oracle_from_loaded

pytestmark = pytest.mark.gpu
pytest.importorskip("transformers")


def _request(model, s, lens, n_suf, seed, dtype):
    rng = np.random.default_rng(seed)
    N = sum(lens)
    tok = rng.integers(0, s.vocab, N + n_suf + 1)
    cs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    Kc, Vc = engine_chunk_caches(model, s, tok, cs)
    req = types.SimpleNamespace(n_ctx=N, n_suffix=n_suf, n_total=N + n_suf)
    return tok, cs, round_to(Kc, dtype), round_to(Vc, dtype), req


def _handoff_logits(model, res, tok, N, n_suf):
    Ke = C.library_k_to_engine(torch.from_numpy(res["K"]).double()).numpy()
    return H.decode_with_cache(model, Ke, res["V"], tok[N + n_suf], N + n_suf)


def test_checkpoint_f32_blend_matches_oracle_and_engine(P, tmp_path):
    model = H.make_model(7, kind="mistral")
    model.save_pretrained(str(tmp_path), max_shard_size="150KB")
    s, mw = C.load(str(tmp_path), "f32", "cuda")
    sc, mc = C.load(str(tmp_path), "f32", "cpu")
    m = oracle_from_loaded(sc, mc)
    lens, n_suf = [40, 33, 27], 6
    tok, cs, Kc, Vc, req = _request(model, s, lens, n_suf, 3, "f32")
    N, T = req.n_ctx, req.n_total
    pos = np.arange(T)
    ks = O.schedule(0.3, N, s.n_layers)
    ora = O.blend_forward(m, tok[:T], pos, cs, n_suf, Kc, Vc, ks)
    res = run_blend(P, s, "f32", 0, req, tok[:T], pos, cs, Kc, Vc, ks, force_sel=ora.sel, mw=mw)
    for i in range(s.n_layers):
        assert rel_err(res["K"][i], ora.K[i]) < 1e-4 and rel_err(res["V"][i], ora.V[i]) < 1e-4, i
    assert rel_err(res["h"], ora.h_final) < 1e-4
    full = H.prefill(model, tok[:T + 1])
    r1 = run_blend(P, s, "f32", 0, req, tok[:T], pos, cs, Kc, Vc, O.schedule(1.0, N, s.n_layers), mw=mw,
                   ctx=res["ctx"])
    assert rel_err(_handoff_logits(model, r1, tok, N, n_suf), full["logits"][-1]) < 1e-4


def test_checkpoint_bf16_blend_free_run(P, tmp_path):
    """bf16 on a checkpoint with the small test shape (hd 128, GQA 4, tcgen05 GEMMs and attention): free-running
    selection inside the bf16 deviation band of the oracle's (band_check), recomputed rows of K/V and the
    output rows in replay within the bf16 tolerance; the r = 1 hand-off reproduces the engine's full-prefill
    logits to bf16 accuracy."""
    model = H.make_model(8, n_layers=3, d=1024, n_q=8, n_kv=2, hd=128, ff=2816, vocab=1000, theta=10000.0,
                         eps=1e-5, kind="llama")
    model.save_pretrained(str(tmp_path))
    s, mw = C.load(str(tmp_path), "bf16", "cuda")
    sc, mc = C.load(str(tmp_path), "bf16", "cpu")
    m = oracle_from_loaded(sc, mc)
    lens, n_suf = [300, 211, 157], 9
    tok, cs, Kc, Vc, req = _request(model, s, lens, n_suf, 4, "bf16")
    N, T = req.n_ctx, req.n_total
    pos = np.arange(T)
    ks = O.schedule(0.15, N, s.n_layers)
    ora = O.blend_forward(m, tok[:T], pos, cs, n_suf, Kc, Vc, ks)
    res = run_blend(P, s, "bf16", 0, req, tok[:T], pos, cs, Kc, Vc, ks, mw=mw)
    for i in range(1, s.n_layers):
        ok, flips, band = band_check(res["sel"][i], res["dev"][i][:len(ora.cand[i])], ora.dev[i], ora.cand[i], ks[i])
        assert ok, f"layer {i}: {flips} flips outside the band {band}"
    rep = run_blend(P, s, "bf16", 0, req, tok[:T], pos, cs, Kc, Vc, ks, force_sel=ora.sel, mw=mw, ctx=res["ctx"])
    for i in range(1, s.n_layers):
        rows = np.concatenate([ora.sel[i], np.arange(N, T)])
        assert rel_err(rep["K"][i][rows], ora.K[i][rows]) < 2e-2, f"K layer {i}"
        assert rel_err(rep["V"][i][rows], ora.V[i][rows]) < 2e-2, f"V layer {i}"
    assert rel_err(rep["h"], ora.h_final) < 2e-2
    full = H.prefill(model, tok[:T + 1])
    r1 = run_blend(P, s, "bf16", 0, req, tok[:T], pos, cs, Kc, Vc, O.schedule(1.0, N, s.n_layers), mw=mw,
                   ctx=res["ctx"])
    assert rel_err(_handoff_logits(model, r1, tok, N, n_suf), full["logits"][-1]) < 3e-2
