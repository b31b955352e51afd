"""Test-side Hugging Face reference model: a seeded random-init Mistral/Llama model from `transformers`, saved as
a safetensors checkpoint (the format checkpoint.py reads) and run by transformers' own code as the independent
reference for the loader, for the oracle's decoder block (R-model) and for the KV hand-off to an engine
(P:2748). Nothing here is CacheBlend arithmetic; transformers implements half-split RoPE and its own attention."""
from __future__ import annotations

import math
from typing import Dict, List

import numpy as np
import torch


def make_model(seed: int, n_layers=3, d=64, n_q=4, n_kv=2, hd=16, ff=128, vocab=256, theta=5000.0, eps=1e-6,
               kind="mistral"):
    """Random-init model in fp32 with the synth recipe's scales (linear u/sqrt(fan_in), gains 1 + 0.1u, embed u),
    so every term of the block carries weight (HF's 0.02-std init would make the residual stream dominate)."""
    import transformers as T
    kw = dict(vocab_size=vocab, hidden_size=d, intermediate_size=ff, num_hidden_layers=n_layers,
              num_attention_heads=n_q, num_key_value_heads=n_kv, head_dim=hd, rope_theta=theta, rms_norm_eps=eps,
              max_position_embeddings=8192, tie_word_embeddings=False, attn_implementation="eager")
    if kind == "mistral":
        cfg = T.MistralConfig(sliding_window=None, **kw)
        model = T.MistralForCausalLM(cfg)
    else:
        cfg = T.LlamaConfig(**kw)
        model = T.LlamaForCausalLM(cfg)
    g = torch.Generator().manual_seed(seed)
    with torch.no_grad():
        for name, p in model.named_parameters():
            u = torch.rand(p.shape, generator=g, dtype=torch.float64) * 2 - 1
            if name.endswith("norm.weight"):
                p.copy_(1 + 0.1 * u)
            elif "embed_tokens" in name:
                p.copy_(u)
            else:
                p.copy_(u / math.sqrt(p.shape[1]))
    return model.float().eval()


@torch.no_grad()
def prefill(model, tok: np.ndarray, pos0: int = 0) -> Dict[str, np.ndarray]:
    """transformers' forward over `tok` at positions pos0.. : per-layer K (half-split RoPE order, as the engine
    stores it) and V as [L][T][n_kv][hd], the residual stream after every layer [L][T][d] (pre final norm),
    and the logits [T][vocab]."""
    ids = torch.from_numpy(np.asarray(tok, np.int64))[None]
    pid = torch.arange(pos0, pos0 + ids.shape[1])[None]
    outs: List[torch.Tensor] = []
    hooks = [l.register_forward_hook(lambda m, i, o: outs.append((o[0] if isinstance(o, tuple) else o)[0].clone()))
             for l in model.model.layers]
    try:
        o = model(ids, position_ids=pid, use_cache=True)
    finally:
        for h in hooks:
            h.remove()
    pk = o.past_key_values
    K = np.stack([pk.layers[i].keys[0].permute(1, 0, 2).double().numpy() for i in range(len(outs))])
    V = np.stack([pk.layers[i].values[0].permute(1, 0, 2).double().numpy() for i in range(len(outs))])
    return dict(K=K, V=V, h=np.stack([x.double().numpy() for x in outs]), logits=o.logits[0].double().numpy())


@torch.no_grad()
def decode_with_cache(model, K: np.ndarray, V: np.ndarray, next_tok: int, pos: int) -> np.ndarray:
    """The engine side of the hand-off: one decode step of `next_tok` at position `pos` over a KV cache
    K, V [L][T][n_kv][hd] given in the engine's (half-split) order. Returns the logits [vocab]."""
    from transformers import DynamicCache
    cache = DynamicCache()
    for i in range(K.shape[0]):
        k = torch.from_numpy(np.ascontiguousarray(K[i], np.float32)).permute(1, 0, 2)[None]
        v = torch.from_numpy(np.ascontiguousarray(V[i], np.float32)).permute(1, 0, 2)[None]
        cache.update(k, v, i)
    o = model(torch.tensor([[int(next_tok)]]), position_ids=torch.tensor([[int(pos)]]), past_key_values=cache,
              use_cache=True)
    return o.logits[0, -1].double().numpy()
