"""CacheBlend oracle: plain, slow, fp64 CPU implementation of the blend hot path.

*** TEST INFRASTRUCTURE ONLY. ***  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module. The
product path (`paper_2405_16444_b200`) never imports it and shares no code with it.

Every function follows PAPER.md (`P:<line>`, /root/reference/PAPER.md) in the paper's
order and notation; where the paper is silent or garbled the reading is SURVEY.md
§8(c) R1..R14, restated in DESIGN.md "Readings". Arithmetic is numpy float64; a
matmul (`@`) is the only library primitive used as a step. No blocking, fusion or
reordering beyond what the definitions state.

Notation (Table "Summary of terminology"): i = layer index, j = token index,
KV^pre = precomputed chunk caches, KV^new = CacheBlend-updated cache,
Delta_kv = per-token KV deviation. Positions: g = global, l = chunk-local.

Parity pins (tests/test_oracle_*.py) — every function below is pinned by at least
one check that does not restate its formula:
  rope_*            unit circle, hand values cos 1/sin 1, m=0 identity, norm,
                    relative-position invariance
  realign           R(g-l)R(l)k = R(g)k (closed form)
  rms_norm, attention, mlp, full_prefill
                    torch.nn.functional reference (library routine) in fp64,
                    constant-key closed form, single-key closed form, causality
  kv_deviation      identity -> 0, single-coordinate delta -> delta^2, rotation invariance
  select_hkvd       brute force + SPEC examples S:272-274 (golden)
  schedule          golden S:263-265 + closed form R4/R5
  blend_forward     r=1 -> full prefill; r=0 -> realigned cache; single chunk -> prefix
                    reuse; nesting, untouched entries bitwise, MAC ratio.
  blend_replay_rows equals blend_forward(force_sel) on the rows it returns (to fp64 rounding: the
                    same functions on row subsets), tests/test_oracle_blend.py.
  Intermediate-r selected sets/values: the oracle IS the definition ("parity unpinned"
  beyond the invariants above; SURVEY §8(c) last row).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

F64 = np.float64


# ---------------------------------------------------------------------------------------
# RoPE (Appendix "N-dimensional positional recovery"; footnote P:208-211)
# ---------------------------------------------------------------------------------------
def rope_thetas(head_dim: int, base: float) -> np.ndarray:
    """theta_i = base^(-2i/d), i = 0..d/2-1.  P:2541 prints 10000^{-2id}; reading R8."""
    i = np.arange(head_dim // 2, dtype=F64)
    return np.power(F64(base), -2.0 * i / head_dim)


def rope_rotate(x: np.ndarray, m: np.ndarray, base: float) -> np.ndarray:
    """R^d_{Theta,m} x for x[..., d] at positions m[...] (broadcast over x's leading dims).

    R is block diagonal with 2x2 blocks [[cos m th_i, -sin m th_i], [sin m th_i, cos m th_i]]
    acting on the pair (x[2i], x[2i+1]) (interleaved pairing, reading R9).
    The product is written out per block; angles are formed in fp64."""
    x = np.asarray(x, dtype=F64)
    d = x.shape[-1]
    th = rope_thetas(d, base)
    m = np.asarray(m, dtype=F64)
    m = m.reshape(m.shape + (1,) * (x.ndim - 1 - m.ndim))      # m indexes x's leading dims
    ang = m[..., None] * th                                   # [..., d/2]
    c, s = np.cos(ang), np.sin(ang)
    x0, x1 = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = c * x0 - s * x1
    out[..., 1::2] = s * x0 + c * x1
    return out


def rope_rotate_half(x: np.ndarray, m: np.ndarray, base: float) -> np.ndarray:
    """The half-split RoPE convention of common checkpoints (SURVEY §8(c) R9 "the half-split variant";
    N3 real-checkpoint loading): the pair (x[i], x[i + d/2]) is rotated by m theta_i, i.e.
    y = x cos + rotate_half(x) sin with rotate_half([a, b]) = [-b, a] over the two halves. Test
    reference for the loader-side conversion to the paper's interleaved pairing (R9)."""
    x = np.asarray(x, dtype=F64)
    d = x.shape[-1]
    th = rope_thetas(d, base)
    m = np.asarray(m, dtype=F64)
    m = m.reshape(m.shape + (1,) * (x.ndim - 1 - m.ndim))
    ang = m[..., None] * th
    c, s = np.cos(ang), np.sin(ang)
    a, b = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([c * a - s * b, s * a + c * b], axis=-1)


def realign(k_cached: np.ndarray, src_pos: np.ndarray, dst_pos: np.ndarray, base: float) -> np.ndarray:
    """Positional recovery (footnote P:208-211): K_hat[t] = R(dst_t - src_t) K_cached[t].

    K_cached[t] was encoded at src_t (chunk-local l; 0 = stored without position, R11);
    R(a)R(b) = R(a+b) for the block rotation, so one rotation by g-l moves it to g.
    k_cached: [T][n_kv][hd]; positions [T]."""
    delta = np.asarray(dst_pos, dtype=F64) - np.asarray(src_pos, dtype=F64)
    return rope_rotate(k_cached, delta, base)


# ---------------------------------------------------------------------------------------
# Transformer pieces (Llama/Mistral-style decoder; the paper never states the block,
# SURVEY §8(c) "Model"; attention form softmax(q^T K / sqrt d) P:2068)
# ---------------------------------------------------------------------------------------
class MacCounter:
    """Counts multiply-accumulates of every matmul (S:283/S:316 MAC proportionality pin)."""

    def __init__(self):
        self.macs = 0

    def mm(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        self.macs += int(a.shape[0]) * int(a.shape[1]) * int(b.shape[1])
        return a @ b


def rms_norm(h: np.ndarray, gain: np.ndarray, eps: float) -> np.ndarray:
    """x = h / sqrt(mean(h^2) + eps) * gain, per row."""
    h = np.asarray(h, dtype=F64)
    return h / np.sqrt(np.mean(h * h, axis=-1, keepdims=True) + eps) * np.asarray(gain, F64)


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def causal_attention(q: np.ndarray, q_pos: np.ndarray, k: np.ndarray, v: np.ndarray,
                     k_pos: np.ndarray, mc: Optional[MacCounter] = None, threads: int = 1) -> np.ndarray:
    """Forward attention of query rows over ALL given keys, masked by original position.

    q [R][n_q][hd] (rotated), k/v [T][n_kv][hd] (k rotated), mask: key visible iff
    k_pos <= q_pos (causal by original position; the selected tokens attend to "all
    other tokens"). GQA: q head h reads kv head h // (n_q / n_kv).
    Returns [R][n_q*hd]. `threads` > 1 evaluates the (independent) heads on a thread pool;
    every head's arithmetic is the same either way."""
    R, n_q, hd = q.shape
    n_kv = k.shape[1]
    grp = n_q // n_kv
    visible = np.asarray(k_pos)[None, :] <= np.asarray(q_pos)[:, None]      # [R][T]
    out = np.zeros((R, n_q, hd), dtype=F64)

    def head(h):
        g = h // grp
        s = (q[:, h, :] @ k[:, g, :].T) / math.sqrt(hd)                     # [R][T]
        s[~visible] = -np.inf
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)                                                    # p (unnormalised)
        s /= s.sum(axis=1, keepdims=True)
        out[:, h, :] = s @ v[:, g, :]

    if mc is not None:
        mc.macs += n_q * 2 * R * int(visible.sum(axis=1).mean() if R else 0) * hd
    if threads > 1 and n_q > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(threads, n_q)) as ex:
            list(ex.map(head, range(n_q)))
    else:
        for h in range(n_q):
            head(h)
    return out.reshape(R, n_q * hd)


def mlp(x: np.ndarray, w: Dict[str, np.ndarray], mc: Optional[MacCounter] = None) -> np.ndarray:
    """SwiGLU MLP: W_down (silu(x W_gate^T) * x W_up^T)."""
    mm = mc.mm if mc is not None else (lambda a, b: a @ b)
    g = mm(x, w["wg"].T)
    u = mm(x, w["wu"].T)
    return mm(silu(g) * u, w["wd"].T)


def _w64(w: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
    return {k: np.asarray(v, dtype=F64) for k, v in w.items()}


@dataclass
class Model:
    """Oracle-side model: shape + per-layer weight dicts (fp64 copies of the stored values)."""
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    rope_theta: float
    rms_eps: float
    embed: np.ndarray
    layers: List[Dict[str, np.ndarray]]

    @staticmethod
    def build(shape, embed, layers) -> "Model":
        return Model(shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads,
                     shape.head_dim, shape.rope_theta, shape.rms_eps,
                     np.asarray(embed, F64), [_w64(w) for w in layers])

    @property
    def kvd(self) -> int:
        return self.n_kv_heads * self.head_dim


def qkv(model: Model, i: int, h_rows: np.ndarray, pos: np.ndarray, mc: Optional[MacCounter] = None,
        need_q: bool = True):
    """x = RMSNorm(h); q = RoPE(x W_q^T, g), k = RoPE(x W_k^T, g), v = x W_v^T."""
    w = model.layers[i]
    mm = mc.mm if mc is not None else (lambda a, b: a @ b)
    R = h_rows.shape[0]
    x = rms_norm(h_rows, w["attn_norm"], model.rms_eps)
    q = None
    if need_q:
        q = rope_rotate(mm(x, w["wq"].T).reshape(R, model.n_q_heads, model.head_dim), pos[:, None],
                        model.rope_theta)
    k = rope_rotate(mm(x, w["wk"].T).reshape(R, model.n_kv_heads, model.head_dim), pos[:, None],
                    model.rope_theta)
    v = mm(x, w["wv"].T).reshape(R, model.n_kv_heads, model.head_dim)
    return q, k, v


def attn_out_mlp(model: Model, i: int, h_rows: np.ndarray, attn: np.ndarray,
                 mc: Optional[MacCounter] = None) -> np.ndarray:
    """h += a W_o^T; h += MLP(RMSNorm(h)) (residual connections)."""
    w = model.layers[i]
    mm = mc.mm if mc is not None else (lambda a, b: a @ b)
    h = h_rows + mm(attn, w["wo"].T)
    return h + mlp(rms_norm(h, w["mlp_norm"], model.rms_eps), w, mc)


# ---------------------------------------------------------------------------------------
# Full prefill (§2 Background P:292-316): the textbook forward, used for chunk
# precompute (KV^pre of each chunk at its local positions) and as the r = 100 % pin.
# ---------------------------------------------------------------------------------------
def full_prefill(model: Model, tok: np.ndarray, pos: np.ndarray, mc: Optional[MacCounter] = None):
    """Returns K [L][T][n_kv][hd] (rotated at pos), V [L][T][n_kv][hd], h [T][d]."""
    pos = np.asarray(pos)
    h = model.embed[np.asarray(tok)]
    Ks, Vs = [], []
    for i in range(model.n_layers):
        q, k, v = qkv(model, i, h, pos, mc)
        a = causal_attention(q, pos, k, v, pos, mc)
        h = attn_out_mlp(model, i, h, a, mc)
        Ks.append(k)
        Vs.append(v)
    return np.stack(Ks), np.stack(Vs), h


def precompute_chunk_caches(model: Model, tok: np.ndarray, chunk_starts: Sequence[int]):
    """KV^pre: each chunk prefilled standalone at local positions 0..L_c-1,
    concatenated. K is rotated at the chunk-local positions (BASELINE north_star)."""
    Ks, Vs = [], []
    for c in range(len(chunk_starts) - 1):
        t = np.asarray(tok[chunk_starts[c]:chunk_starts[c + 1]])
        K, V, _ = full_prefill(model, t, np.arange(len(t)))
        Ks.append(K)
        Vs.append(V)
    return np.concatenate(Ks, axis=1), np.concatenate(Vs, axis=1)


# ---------------------------------------------------------------------------------------
# HKVD selection (§3.3)
# ---------------------------------------------------------------------------------------
def kv_deviation(k_new: np.ndarray, v_new: np.ndarray, k_ref: np.ndarray, v_ref: np.ndarray,
                 mode: str = "kv") -> np.ndarray:
    """Delta_kv per token: squared L2 distance between the recomputed
    and the loaded K,V of the token over all kv heads (reading R1: squared L2 over the
    concatenated K and V; 'k' / 'v' restrict to one of them)."""
    dk = np.asarray(k_new, F64) - np.asarray(k_ref, F64)
    dv = np.asarray(v_new, F64) - np.asarray(v_ref, F64)
    n = dk.shape[0]
    dev = np.zeros(n, dtype=F64)
    if mode in ("kv", "k"):
        dev += (dk.reshape(n, dk[0].size if n else 0) ** 2).sum(axis=1)
    if mode in ("kv", "v"):
        dev += (dv.reshape(n, dv[0].size if n else 0) ** 2).sum(axis=1)
    return dev


def select_hkvd(dev: np.ndarray, cand_tok: np.ndarray, k_keep: int) -> np.ndarray:
    """The k_keep candidates with the highest deviation (Insight 1); ties go to
    the lower token index (R6). Returned sorted ascending by token index."""
    order = np.lexsort((np.asarray(cand_tok), -np.asarray(dev, F64)))
    return np.sort(np.asarray(cand_tok)[order[:k_keep]])


def schedule_ratios(ratio: float, n_layers: int) -> List[float]:
    """Gradual-filtering ratios r_1..r_{L-1} (reading R4).

    r_i = r + delta (1 - 2(i-1)/(L-2)), delta = 0.2 min(r, 1-r): r_1 slightly above r, each next
    slightly below the previous, mean exactly r; L = 2 gives [r]."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio out of [0, 1]")
    if n_layers < 1:
        raise ValueError("bad shape")
    delta = 0.2 * min(ratio, 1.0 - ratio)
    out = []
    for i in range(1, n_layers):
        out.append(ratio if n_layers == 2 else ratio + delta * (1.0 - 2.0 * (i - 1) / (n_layers - 2)))
    return out


def schedule(ratio: float, n_ctx: int, n_layers: int) -> List[int]:
    """Per-layer counts k_i = |S_i| (reading R5): k_i = min(N, ceil(r_i N - 1e-9)), kept
    non-increasing so the sets can nest. Layer 0 is the full layer (R2), so k[0] = N."""
    if n_ctx < 0:
        raise ValueError("bad shape")
    ks = [n_ctx]
    for ri in schedule_ratios(ratio, n_layers):
        ki = min(n_ctx, int(math.ceil(ri * n_ctx - 1e-9)))
        ks.append(max(0, min(ki, ks[-1])))
    return ks


# ---------------------------------------------------------------------------------------
# The blend (§3.2 workflow P:150-161, gradual filtering P:284-287, prefill_layer P:2507)
# ---------------------------------------------------------------------------------------
@dataclass
class BlendResult:
    K: np.ndarray                       # KV^new, [L][T][n_kv][hd]
    V: np.ndarray
    sel: List[np.ndarray]               # S_i (token indices, ascending); sel[0] = all context
    dev: List[Optional[np.ndarray]]     # Delta_kv over C_i (aligned with cand[i]); dev[0] = None
    cand: List[np.ndarray]              # C_i
    h_final: np.ndarray                 # h rows of S_{L-1} followed by the suffix rows
    h_layers: List[np.ndarray] = field(default_factory=list)   # h rows after each layer
    macs: int = 0


def blend_layer(model: Model, i: int, h_cand: np.ndarray, cand: np.ndarray, n_ctx: int, n_suf: int,
                k_keep: int, K: np.ndarray, V: np.ndarray, pos: np.ndarray,
                force_sel: Optional[np.ndarray] = None, dev_mode: str = "kv",
                mc: Optional[MacCounter] = None):
    """prefill_layer with check_flag on layer i >= 1, updating K[i], V[i] in place.

    h_cand: h rows of C_i (ascending) followed by the n_suf suffix rows.
    1. mask the input to C_i (+ suffix) and compute Q, K, V only for those rows;
    2. Delta_kv of each candidate against the loaded (realigned) entry (R1);
    3. S_i = top-k_keep of C_i (Insight 1; replaced by force_sel in replay mode, R14);
    4. write the fresh K,V of S_i (+ suffix) into the cache; untouched rows keep KV^pre (R3);
    5. attention of the S_i (+ suffix) queries over all tokens' K,V, W_o, MLP.
    Returns (h rows of S_i + suffix, S_i, dev over C_i)."""
    rows = np.concatenate([cand, n_ctx + np.arange(n_suf)]).astype(np.int64)
    q, k, v = qkv(model, i, h_cand, pos[rows], mc)
    nc = len(cand)
    dev = kv_deviation(k[:nc], v[:nc], K[i][cand], V[i][cand], dev_mode)
    sel = select_hkvd(dev, cand, k_keep) if force_sel is None else np.sort(np.asarray(force_sel))
    slot = np.searchsorted(cand, sel)
    if len(sel) and not np.array_equal(cand[np.minimum(slot, nc - 1)], sel):
        raise ValueError("force_sel is not a subset of the candidates")
    keep = np.concatenate([slot, nc + np.arange(n_suf)]).astype(np.int64)
    K[i][rows[keep]] = k[keep]
    V[i][rows[keep]] = v[keep]
    T = K.shape[1]
    a = causal_attention(q[keep], pos[rows[keep]], K[i], V[i], pos[:T], mc)
    h_new = attn_out_mlp(model, i, h_cand[keep], a, mc)
    return h_new, sel, dev


def blend_forward(model: Model, tok: np.ndarray, pos: np.ndarray, chunk_starts: Sequence[int],
                  n_suf: int, Kc: np.ndarray, Vc: np.ndarray, k_sched: Sequence[int],
                  force_sel: Optional[Sequence[np.ndarray]] = None, dev_mode: str = "kv",
                  count_macs: bool = False, keep_layers: bool = False) -> BlendResult:
    """Whole blend (SURVEY §8(c) algorithm steps 1-5).

    tok, pos: [N + n_suf] (context then suffix); Kc, Vc: [L][N][n_kv][hd] chunk caches with K
    rotated at chunk-local positions; k_sched[i] = |S_i| for i >= 1 (k_sched[0] unused)."""
    tok = np.asarray(tok)
    pos = np.asarray(pos).astype(np.int64)
    N = int(chunk_starts[-1])
    T = N + n_suf
    L = model.n_layers
    mc = MacCounter() if count_macs else None
    loc = np.zeros(N, dtype=np.int64)
    for c in range(len(chunk_starts) - 1):
        loc[chunk_starts[c]:chunk_starts[c + 1]] = np.arange(chunk_starts[c + 1] - chunk_starts[c])

    # 1. realign every layer's cached K from chunk-local to global positions;
    #    V carries no position.  This initialises KV^new.
    K = np.zeros((L, T, model.n_kv_heads, model.head_dim), dtype=F64)
    V = np.zeros_like(K)
    for i in range(L):
        K[i, :N] = realign(Kc[i], loc, pos[:N], model.rope_theta)
        V[i, :N] = np.asarray(Vc[i], F64)

    # 2. layer 0 in full ("perform prefill on the first layer first"; R2). Context rows
    #    keep the realigned cache (layer-0 K/V depend only on the token); suffix rows
    #    have no cache and write their fresh K/V.
    h = model.embed[tok]
    q, k, v = qkv(model, 0, h, pos, mc, need_q=True)
    K[0, N:] = k[N:]
    V[0, N:] = v[N:]
    a = causal_attention(q, pos, K[0], V[0], pos, mc)
    h = attn_out_mlp(model, 0, h, a, mc)
    sel = [np.arange(N)]
    devs: List[Optional[np.ndarray]] = [None]
    cands = [np.arange(N)]
    h_layers = [h.copy()] if keep_layers else []

    # 3. layers 1..L-1: gradual filtering, C_{i+1} = S_i.
    cand = np.arange(N)
    for i in range(1, L):
        fs = None if force_sel is None else force_sel[i]
        h, s, dv = blend_layer(model, i, h, cand, N, n_suf, int(k_sched[i]), K, V, pos, fs,
                               dev_mode, mc)
        cands.append(cand)
        sel.append(s)
        devs.append(dv)
        cand = s
        if keep_layers:
            h_layers.append(h.copy())
    return BlendResult(K, V, sel, devs, cands, h, h_layers, mc.macs if mc else 0)


def attention_probs(q: np.ndarray, q_pos: np.ndarray, k: np.ndarray, k_pos: np.ndarray) -> np.ndarray:
    """The forward attention matrix A: softmax(q k^T / sqrt(hd)) of each query row and q head over all
    given keys, masked by original position (key visible iff k_pos <= q_pos), GQA as causal_attention.
    q [R][n_q][hd] (rotated), k [T][n_kv][hd] (rotated). Returns [n_q][R][T]."""
    R, n_q, hd = q.shape
    grp = n_q // k.shape[1]
    visible = np.asarray(k_pos)[None, :] <= np.asarray(q_pos)[:, None]
    A = np.zeros((n_q, R, k.shape[0]), dtype=F64)
    for h in range(n_q):
        s = (q[:, h, :] @ k[:, h // grp, :].T) / math.sqrt(hd)
        s[~visible] = -np.inf
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        A[h] = p / p.sum(axis=1, keepdims=True)
    return A


def attention_deviation(model: Model, tok: np.ndarray, pos: np.ndarray, chunk_starts: Sequence[int], n_suf: int,
                        Kc: np.ndarray, Vc: np.ndarray, k_sched: Sequence[int],
                        force_sel: Optional[Sequence[np.ndarray]] = None) -> np.ndarray:
    """Attention deviation per layer, Delta_attn(A_i, A_i^full): the L-2 norm of the difference
    between the forward attention matrix of layer i after the blend and after full prefill (reading R16: the
    matrix of the query rows -- the n_suf uncached suffix tokens, the user query of P:2793 -- over every key;
    each side's queries come from its own layer input, i.e. the hidden states its KV produced).
    Returns [L] (layer 0 is exactly 0: its KV and its queries do not depend on cross-chunk attention)."""
    if n_suf < 1:
        raise ValueError("attention deviation needs query (suffix) rows")
    tok, pos = np.asarray(tok), np.asarray(pos).astype(np.int64)
    qpos = pos[-n_suf:]
    res = blend_forward(model, tok, pos, chunk_starts, n_suf, Kc, Vc, k_sched, force_sel=force_sel,
                        keep_layers=True)
    h_full = model.embed[tok]
    out = np.zeros(model.n_layers, dtype=F64)
    for i in range(model.n_layers):
        hb = model.embed[tok[-n_suf:]] if i == 0 else res.h_layers[i - 1][-n_suf:]
        qb = qkv(model, i, hb, qpos)[0]
        qf, kf, vf = qkv(model, i, h_full, pos)
        a_blend = attention_probs(qb, qpos, res.K[i], pos)
        a_full = attention_probs(qf[-n_suf:], qpos, kf, pos)
        out[i] = float(np.sqrt(np.sum((a_blend - a_full) ** 2)))
        h_full = attn_out_mlp(model, i, h_full, causal_attention(qf, pos, kf, vf, pos))
    return out


def blend_replay_rows(tok: np.ndarray, pos: np.ndarray, chunk_starts: Sequence[int], Kc: np.ndarray,
                      Vc: np.ndarray, force_sel: Sequence[np.ndarray], layer_model, embed_rows: np.ndarray,
                      dev_rows_1: Sequence[int] = (), h_rows_last: Optional[Sequence[int]] = None,
                      threads: int = 1, h0: Optional[np.ndarray] = None):
    """The blend of `blend_forward` in replay mode (forced S_i, R14), n_suf = 0, evaluated only on the rows
    the comparison needs -- for full-width models whose full oracle run would take hours.

    Every row of every layer is computed exactly as in `blend_layer` / `blend_forward` (same functions,
    same order); rows whose results cannot reach a compared output are skipped:
    - layer 0 runs its queries only for S_1 plus `dev_rows_1` (layer-0 K/V of context rows are the realigned
      cache, so no other row is needed);
    - layer i >= 1 runs Q, K, V for its candidates C_i = S_{i-1} (C_1 restricted to the rows above), takes
      Delta_kv of all of them, writes S_i's fresh K, V (R3) and runs attention + W_o + MLP for S_i;
    - on the last layer attention + MLP run only for `h_rows_last` (a subset of S_{L-1}; all when None).
    layer_model(i) returns a `Model` whose layers[i] holds layer i's weights (fp64); embed_rows[t] is the
    embedding row of token t (embed[tok[t]]). h0: layer 0's output for every context row, when the caller
    already has it (layer 0 does not depend on the selections; it is then not recomputed). Returns dict(K,
    V [L][N][n_kv][hd] (KV^new), dev {i: (rows, Delta_kv)}, h_rows (token ids), h (their final hidden
    rows))."""
    tok = np.asarray(tok)
    pos = np.asarray(pos).astype(np.int64)
    N = int(chunk_starts[-1])
    L = len(Kc)
    loc = np.zeros(N, dtype=np.int64)
    for c in range(len(chunk_starts) - 1):
        loc[chunk_starts[c]:chunk_starts[c + 1]] = np.arange(chunk_starts[c + 1] - chunk_starts[c])
    m0 = layer_model(0)
    n_kv, hd, theta = m0.n_kv_heads, m0.head_dim, m0.rope_theta
    K = np.zeros((L, N, n_kv, hd), dtype=F64)
    V = np.zeros_like(K)
    for i in range(L):  # 1. realign
        K[i] = realign(Kc[i], loc, pos[:N], theta)
        V[i] = np.asarray(Vc[i], F64)
    sel = [np.arange(N)] + [np.sort(np.asarray(s, np.int64)) for s in force_sel[1:L]]
    rows = np.arange(N) if L == 1 else np.union1d(sel[1], np.asarray(dev_rows_1, np.int64))
    if L == 1 and h_rows_last is not None:
        rows = np.sort(np.asarray(h_rows_last, np.int64))
    # 2. layer 0 on `rows`: queries over the realigned cache, W_o, MLP (R2)
    if h0 is not None:
        h = np.asarray(h0, F64)[rows]
    else:
        h = np.asarray(embed_rows, F64)[rows]
        q, _, _ = qkv(m0, 0, h, pos[rows])
        a = causal_attention(q, pos[rows], K[0], V[0], pos[:N], threads=threads)
        h = attn_out_mlp(m0, 0, h, a)
    del m0
    dev = {}
    # 3. layers 1..L-1 in replay
    for i in range(1, L):
        mi = layer_model(i)
        q, k, v = qkv(mi, i, h, pos[rows])
        dev[i] = (rows.copy(), kv_deviation(k, v, K[i][rows], V[i][rows]))
        slot = np.searchsorted(rows, sel[i])
        if len(sel[i]) and not np.array_equal(rows[np.minimum(slot, len(rows) - 1)], sel[i]):
            raise ValueError("force_sel is not a subset of the candidates")
        K[i][sel[i]] = k[slot]
        V[i][sel[i]] = v[slot]
        qsel = sel[i] if (i < L - 1 or h_rows_last is None) else np.sort(np.asarray(h_rows_last, np.int64))
        qs = np.searchsorted(rows, qsel)
        a = causal_attention(q[qs], pos[qsel], K[i], V[i], pos[:N], threads=threads)
        h = attn_out_mlp(mi, i, h[qs], a)
        rows = qsel
    return dict(K=K, V=V, dev=dev, h_rows=rows, h=h)


def full_prefill_macs(model: Model, tok, pos) -> int:
    mc = MacCounter()
    full_prefill(model, tok, pos, mc)
    return mc.macs


# ---------------------------------------------------------------------------------------
# Loading controller (§6 "Loading Controller", P:2693-2705 and its two footnotes)
# ---------------------------------------------------------------------------------------
def t_recompute(ratio: float, prefill_ms: float) -> float:
    """Recompute delay estimator: T_recompute(r%, LLM, L) = r% x Prefill(LLM, L) (footnote),
    Prefill profiled offline. Per layer (P:2666-2670 compare one layer's recompute with one layer's load)."""
    return float(ratio) * float(prefill_ms)


def t_load(kv_bytes_per_token: float, n_tokens: int, bytes_per_ms: float) -> float:
    """Loading delay estimator: T_load = PerTokenKVSize(LLM) x L / Throughput(storage_device) (footnote,
    P:2696), for one layer's KV."""
    return float(kv_bytes_per_token) * int(n_tokens) / float(bytes_per_ms)


def controller_ratio(prefill_ms: float, load_ms: float, r_min: float = 0.15) -> float:
    """Pick r% with T_recompute(r%) = T_load, then take max(r%, r*%) with r* = 15 %; a
    ratio is at most 100 %."""
    r_eq = float(load_ms) / float(prefill_ms)
    return min(1.0, max(r_eq, float(r_min)))


def controller_pick_device(prefill_ms: float, load_ms: Sequence[float], cost: Sequence[float],
                           r_fixed: float = 0.15) -> int:
    """The cheapest storage device whose loading delay is hidden by the fixed-ratio recompute,
    T_recompute(r_fixed) >= T_load; ties -> the earlier device; -1 if none qualifies."""
    best = -1
    for d in range(len(load_ms)):
        if t_recompute(r_fixed, prefill_ms) >= load_ms[d] and (best < 0 or cost[d] < cost[best]):
            best = d
    return best


# ---------------------------------------------------------------------------------------
# Hand-off to a paged decode cache ("the fused KV cache is input into the LLM inference
# engine"; vLLM pages KV in fixed-size blocks)
# ---------------------------------------------------------------------------------------
def kv_to_paged(kv: np.ndarray, block_table: Sequence[int], block_size: int, n_pages: int) -> np.ndarray:
    """kv [L][T][n_kv][hd] -> pages [L][n_pages][block_size][n_kv][hd]: token t at page
    block_table[t // block_size], slot t % block_size. Unwritten slots are NaN."""
    L, T = kv.shape[:2]
    out = np.full((L, n_pages, block_size) + kv.shape[2:], np.nan, dtype=kv.dtype)
    for t in range(T):
        out[:, block_table[t // block_size], t % block_size] = kv[:, t]
    return out
