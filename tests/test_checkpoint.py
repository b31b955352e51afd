"""Checkpoint loading: the safetensors reader against the `safetensors` library, and the
loaded weights run through the fp64 oracle against `transformers`' own Mistral/Llama forward (half-split RoPE,
its own attention and norms). The second test pins the loader's stacking and RoPE permutation, config.json
parsing (theta, eps, GQA), and the oracle's decoder block (R-model) to an implementation that shares nothing
with either. Also the KV hand-off: the oracle's blended KV, converted back to the engine's order,
drives a transformers decode step; at r = 1 it reproduces full prefill's next-token logits."""
import json
import os
import struct

import numpy as np
import pytest
import torch

from oracle import cacheblend_oracle as O
from paper_2405_16444_b200 import checkpoint as C
from tests import hf_model as H
from tests.helpers import rel_err

pytest.importorskip("transformers")


def oracle_from_loaded(s, mw) -> O.Model:
    layers = []
    for w in mw.layers:
        qkv = w["w_qkv"].double().numpy()
        gu = w["w_gate_up"].double().numpy()
        layers.append(dict(wq=qkv[:s.qd], wk=qkv[s.qd:s.qd + s.kvd], wv=qkv[s.qd + s.kvd:],
                           wo=w["w_o"].double().numpy(), wg=gu[:s.d_ff], wu=gu[s.d_ff:],
                           wd=w["w_down"].double().numpy(), attn_norm=w["attn_norm"].double().numpy(),
                           mlp_norm=w["mlp_norm"].double().numpy()))
    return O.Model.build(s, mw.embed.double().numpy(), layers)


@pytest.fixture(scope="module", params=["mistral", "llama"])
def hf(request, tmp_path_factory):
    model = H.make_model(5, kind=request.param)
    d = tmp_path_factory.mktemp(request.param)
    model.save_pretrained(str(d), max_shard_size="150KB")  # sharded: exercises the index file
    return model, str(d)


def test_reader_matches_safetensors_library(hf, tmp_path):
    from safetensors import safe_open
    model, d = hf
    ck = C.Checkpoint(d)
    assert os.path.exists(os.path.join(d, "model.safetensors.index.json")) and len(set(ck.where.values())) > 1
    for name, fname in ck.where.items():
        with safe_open(os.path.join(d, fname), "pt") as f:
            assert torch.equal(ck.tensor(name), f.get_tensor(name)), name
    ck.close()
    import copy
    copy.deepcopy(model).to(torch.bfloat16).save_pretrained(str(tmp_path))  # one file, bf16
    ck = C.Checkpoint(str(tmp_path))
    with safe_open(os.path.join(str(tmp_path), "model.safetensors"), "pt") as f:
        for name in f.keys():
            t = ck.tensor(name)
            assert t.dtype == torch.bfloat16 and torch.equal(t, f.get_tensor(name)), name
    ck.close()


def test_loaded_model_matches_transformers(hf):
    """Oracle full prefill (interleaved RoPE, fp64) on the loaded weights == transformers' fp32 forward of the
    checkpoint: every layer's residual stream and V, and K after converting back to the half-split order."""
    model, d = hf
    s, mw = C.load(d, "f32", "cpu")
    cfg = model.config
    assert (s.n_layers, s.d_model, s.n_q_heads, s.n_kv_heads, s.head_dim, s.d_ff, s.vocab) == (
        cfg.num_hidden_layers, cfg.hidden_size, cfg.num_attention_heads, cfg.num_key_value_heads, cfg.head_dim,
        cfg.intermediate_size, cfg.vocab_size)
    assert s.rope_theta == 5000.0 and s.rms_eps == 1e-6
    m = oracle_from_loaded(s, mw)
    tok = np.random.default_rng(1).integers(0, s.vocab, 70)
    for pos0 in (0, 1000):
        ref = H.prefill(model, tok, pos0)
        K, V, h = O.full_prefill(m, tok, np.arange(len(tok)) + pos0)
        for i in range(s.n_layers):
            assert rel_err(C.library_k_to_engine(torch.from_numpy(K[i])).numpy(), ref["K"][i]) < 1e-5, f"K {i}"
            assert rel_err(V[i], ref["V"][i]) < 1e-5, f"V {i}"
        assert rel_err(h, ref["h"][-1]) < 1e-5  # the residual stream after the last layer (h_final)
    # the residual stream after each earlier layer: the oracle on the model truncated to layers 0..i
    import dataclasses
    for i in range(s.n_layers - 1):
        si = dataclasses.replace(s, n_layers=i + 1)
        mi = O.Model.build(si, m.embed, m.layers[:i + 1])
        _, _, hi = O.full_prefill(mi, tok, np.arange(len(tok)))
        assert rel_err(hi, H.prefill(model, tok)["h"][i]) < 1e-5, f"h after layer {i}"


def engine_chunk_caches(model, s, tok, cs):
    """Each chunk prefilled alone by the engine (transformers) at positions 0..len-1; K converted to the
    library's interleaved order (checkpoint.engine_k_to_library)."""
    N = int(cs[-1])
    Kc = np.zeros((s.n_layers, N, s.n_kv_heads, s.head_dim))
    Vc = np.zeros_like(Kc)
    for c in range(len(cs) - 1):
        r = H.prefill(model, tok[cs[c]:cs[c + 1]])
        Kc[:, cs[c]:cs[c + 1]] = C.engine_k_to_library(torch.from_numpy(r["K"])).numpy()
        Vc[:, cs[c]:cs[c + 1]] = r["V"]
    return Kc, Vc


def test_blended_kv_drives_engine_decode(hf):
    """The hand-off: the oracle blend over chunk caches that the engine (transformers) produced, K
    converted to the library's order on the way in and back on the way out, then one transformers decode
    step over the blended cache. r = 1 recomputes every token, so the logits equal full prefill's. Sanity
    check of the method on these random-weight models (not a quality claim, which needs trained weights):
    the next-token logit error against full prefill falls as r grows (full reuse r = 0 worst), the trend the
    paper reports for the attention deviation (Fig. ca_reduction)."""
    model, d = hf
    s, mw = C.load(d, "f32", "cpu")
    m = oracle_from_loaded(s, mw)
    rng = np.random.default_rng(2)
    lens, n_suf = [24, 31, 18], 5
    N = sum(lens)
    tok = rng.integers(0, s.vocab, N + n_suf + 1)
    cs = np.concatenate([[0], np.cumsum(lens)])
    Kc, Vc = engine_chunk_caches(model, s, tok, cs)
    full = H.prefill(model, tok[:N + n_suf + 1])
    err = []
    for ratio in (0.0, 0.15, 0.5, 1.0):
        ks = O.schedule(ratio, N, s.n_layers)
        ora = O.blend_forward(m, tok[:N + n_suf], np.arange(N + n_suf), cs, n_suf, Kc, Vc, ks)
        Ke = C.library_k_to_engine(torch.from_numpy(np.asarray(ora.K))).numpy()
        logits = H.decode_with_cache(model, Ke, np.asarray(ora.V), tok[N + n_suf], N + n_suf)
        err.append(rel_err(logits, full["logits"][-1]))
    assert err[-1] < 1e-5, err
    assert all(a > b for a, b in zip(err, err[1:])), err


def test_loader_errors(hf, tmp_path):
    model, d = hf
    cfg = json.load(open(os.path.join(d, "config.json")))
    with pytest.raises(ValueError, match="sliding_window"):
        C.shape_from_config(dict(cfg, sliding_window=4096))
    assert C.shape_from_config(dict(cfg, sliding_window=4096), max_context=4096).n_layers == cfg["num_hidden_layers"]
    with pytest.raises(ValueError, match="scaled RoPE"):
        C.shape_from_config(dict(cfg, rope_scaling={"type": "linear", "factor": 2.0}))
    with pytest.raises(ValueError, match="hidden_act"):
        C.shape_from_config(dict(cfg, hidden_act="gelu"))
    legacy = {k: v for k, v in cfg.items() if k != "rope_parameters"}
    assert C.shape_from_config(dict(legacy, rope_theta=1e6)).rope_theta == 1e6
    # a tensor whose shape disagrees with config.json, and a missing one
    bad = dict(cfg, intermediate_size=cfg["intermediate_size"] * 2)
    import shutil
    d2 = str(tmp_path / "bad")
    shutil.copytree(d, d2)
    json.dump(bad, open(os.path.join(d2, "config.json"), "w"))
    with pytest.raises(ValueError, match="gate_proj"):
        C.load(d2, "f32", "cpu")
    idx = json.load(open(os.path.join(d, "model.safetensors.index.json")))
    idx["weight_map"].pop("model.layers.1.mlp.up_proj.weight")
    json.dump(cfg, open(os.path.join(d2, "config.json"), "w"))
    json.dump(idx, open(os.path.join(d2, "model.safetensors.index.json"), "w"))
    with pytest.raises(KeyError, match="up_proj"):
        C.load(d2, "f32", "cpu")
    # truncated files
    p = str(tmp_path / "t.safetensors")
    with open(p, "wb") as f:
        f.write(struct.pack("<Q", 1000) + b"{}")
    with pytest.raises(ValueError, match="header length"):
        C.SafetensorsFile(p)
    hdr = json.dumps({"x": {"dtype": "F32", "shape": [4], "data_offsets": [0, 16]}}).encode()
    with open(p, "wb") as f:
        f.write(struct.pack("<Q", len(hdr)) + hdr + b"\0" * 8)
    with pytest.raises(ValueError, match="outside the file"):
        C.SafetensorsFile(p)
