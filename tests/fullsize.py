"""Full-width parity at the BASELINE.json configs (1: Mistral-7B 6x512, 2: Yi-34B 8x1024 at 5/15/30/50 %,
3: Llama-70B 10x1024, 4: batched variable-length requests) -- shared by tests/test_gpu_configs.py and the
head-parallel loopback tests.

Every oracle input comes from the seeded generators (synth/), never from the CUDA path:
- weights: the counter-RNG recipe (`W.layer_weights`), regenerated on the host layer by layer;
- chunk caches: random-cache mode (`W.random_cache`, statistically like real K/V: std ~0.58) -- a full-width
  fp64 precompute of every chunk would take hours;
- replay selections: a seeded nested recipe (`W.nested_selection`) with the config's k_i, passed to BOTH sides
  as force_sel (R14 replay mode).
The model is the configuration's full width at truncated depth (`L_T` layers: layer 0, the check layer 1 and
one gradual-filtering layer 2), with the full-depth schedule's k_1, k_2, so every GEMM / attention / top-k
launch has the shape it has inside the full blend. Layer 0 runs over all N rows on both sides, so the oracle's
layer-1 Delta_kv exists for every token and the GPU's free-running S_1 is compared with the oracle's own top-k.

Tolerances (reading R13, restated per row):
- fresh K/V rows (S_i): per (token, kv head) relative L2 error <= KV_TOL (2^-7, two bf16 roundings);
- untouched K rows: |g - o| <= 2^-8 |o| + 1e-5 max|row| elementwise (bf16 rounding of an fp32 rotation);
  untouched V rows bitwise the cache;
- Delta_kv: per candidate |g - o| <= DEV_TOL * o;
- final h rows: per row relative L2 <= H_TOL;
- free-running selection: S_1 equals the oracle's top-k_1 except tokens whose oracle Delta_kv lies within the
  measured GPU Delta_kv error of the oracle's k_1-th value.
"""
from __future__ import annotations

import dataclasses
import os
import time
from typing import Dict, List

import numpy as np
import torch

from oracle import cacheblend_oracle as O
from synth import workload as W
from tests.helpers import band_check, topk_tokens

DEV = "cuda"
L_T = 3
# Tolerances from the arithmetic (bf16 unit roundoff u = 2^-8): a fresh K/V element carries the rounding of
# its GEMM input (RMSNorm output, <= u relative) and of its own bf16 store (<= u), so 2u per (row, head) in
# L2 -- measured 3.3e-3 on every config (profiles/r02_gpu_configs.log); an injected 1 % error fails it. The
# final h rows (fp32) and Delta_kv inherit the same input roundings: 2u and u respectively (measured 1.7e-3
# and 3.2e-4).
KV_TOL = 2.0 ** -7
H_TOL = 2.0 ** -7
DEV_TOL = 2.0 ** -8
SEED = 1
THREADS = min(16, os.cpu_count() or 1)

# name -> (model, chunk lengths, ratio)
CONFIGS = {
    "mistral15": ("mistral-7b", [512] * 6, 0.15),
    "yi05": ("yi-34b", [1024] * 8, 0.05),
    "yi15": ("yi-34b", [1024] * 8, 0.15),
    "yi30": ("yi-34b", [1024] * 8, 0.30),
    "yi50": ("yi-34b", [1024] * 8, 0.50),
    "llama15": ("llama-70b", [1024] * 10, 0.15),
}


def batched_requests() -> List[W.Request]:
    """BASELINE config 5 (64 Mistral-shape requests of 4-8 chunks x 256-1024 tokens): the two extreme
    shapes (4 x 256, 8 x 1024) plus the first two requests of the config's own seeded list (ragged chunk
    lengths)."""
    reqs = W.config_requests("batched", SEED)
    return [W.Request([256] * 4, 0, 4001, 0.15), W.Request([1024] * 8, 0, 4002, 0.15), reqs[0], reqs[1]]


@dataclasses.dataclass
class Case:
    name: str
    full: W.ModelShape        # the configuration's model (full depth)
    s: W.ModelShape           # truncated depth, full width
    req: W.Request
    seed: int                 # weights (counter-RNG recipe); the request's own seed draws tokens and caches
    tok: np.ndarray
    pos: np.ndarray
    cs: np.ndarray
    ks_full: List[int]
    ks: List[int]             # first L_T entries of ks_full
    S: List[np.ndarray]       # forced (replay) selections
    h_last: np.ndarray        # S_{L-1} rows whose final h the oracle computes
    Kc: np.ndarray            # host chunk caches [L_T][N][n_kv][hd] (stored bf16 values)
    Vc: np.ndarray

    @property
    def N(self) -> int:
        return self.req.n_ctx


def make_case(name: str, model: str, lens, ratio: float, seed: int = SEED, n_h: int = 192,
              req_seed: int = None) -> Case:
    full = W.MODELS[model]
    s = dataclasses.replace(full, n_layers=L_T)
    rs = seed if req_seed is None else req_seed
    req = W.Request(list(lens), 0, rs, ratio)
    N = req.n_ctx
    ks_full = O.schedule(ratio, N, full.n_layers)
    ks = ks_full[:L_T]
    S = W.nested_selection(rs, N, ks)
    h_last = S[-1][W.sample_rows(rs, 0x7A, len(S[-1]), n_h)]
    Kc = np.stack([W.random_cache(s, i, N, rs, "bf16", "k") for i in range(L_T)])
    Vc = np.stack([W.random_cache(s, i, N, rs, "bf16", "v") for i in range(L_T)])
    return Case(name, full, s, req, seed, req.tokens(s.vocab), req.global_positions(), req.chunk_starts(),
                ks_full, ks, S, h_last, Kc, Vc)


def case_for(name: str) -> Case:
    model, lens, ratio = CONFIGS[name]
    return make_case(name, model, lens, ratio)


# ---- oracle (fp64, host) --------------------------------------------------------------------------------
def layer_model(s: W.ModelShape, seed: int):
    """layer_model(i) for O.blend_replay_rows: layer i's weights regenerated from the RNG recipe."""
    def get(i):
        w = W.layer_weights(s, i, seed, "bf16")
        layers = [None] * s.n_layers
        layers[i] = {k: np.asarray(v, np.float64) for k, v in w.items()}
        return O.Model(s.n_layers, s.d_model, s.n_q_heads, s.n_kv_heads, s.head_dim, s.rope_theta, s.rms_eps,
                       np.zeros((1, s.d_model)), layers)
    return get


_H0: Dict[tuple, np.ndarray] = {}
_ORA: Dict[tuple, dict] = {}


def oracle_h0(c: Case) -> np.ndarray:
    """Layer 0's output for every context row (selection-independent; shared by the ratios of a model)."""
    key = (c.s.name, c.seed, c.req.seed, tuple(c.req.chunk_lens))
    if key not in _H0:
        t = time.time()
        emb = W.embed_weights(c.s, c.seed, "bf16")[c.tok]
        r = O.blend_replay_rows(c.tok, c.pos, c.cs, c.Kc[:1], c.Vc[:1], [np.arange(c.N)], layer_model(c.s, c.seed),
                                emb, threads=THREADS)
        _H0[key] = r["h"]
        print(f"[oracle] {c.name}: layer 0 over {c.N} rows in {time.time() - t:.1f} s")
    return _H0[key]


def oracle(c: Case) -> dict:
    """Replay blend of the case (forced S_i) with Delta_kv of every layer-1 token; cached per case."""
    key = (c.name, c.seed, c.req.seed, tuple(c.req.chunk_lens))
    if key not in _ORA:
        h0 = oracle_h0(c)
        t = time.time()
        r = O.blend_replay_rows(c.tok, c.pos, c.cs, c.Kc, c.Vc, c.S, layer_model(c.s, c.seed), None,
                                dev_rows_1=np.arange(c.N), h_rows_last=c.h_last, threads=THREADS, h0=h0)
        print(f"[oracle] {c.name}: layers 1..{L_T - 1} in {time.time() - t:.1f} s")
        _ORA[key] = r
    return _ORA[key]


# ---- GPU -------------------------------------------------------------------------------------------------
def to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=DEV, dtype=dtype)


def gpu_inputs(P, c: Case, shape=None):
    """Device inputs of the case: weights by the library's RNG (cb_gen_fill, pinned bit-exact to synth),
    caches by cb_gen_fill on the same streams as W.random_cache, tokens / positions uploaded."""
    s = shape or c.s
    mw = P.ModelWeights.synth(s, c.seed, "bf16", DEV)
    L, N = s.n_layers, c.N
    k_in = torch.empty(L, N, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=DEV)
    v_in = torch.empty_like(k_in)
    for i in range(L):
        P.api.gen_fill(k_in[i], c.req.seed, W.cache_stream(i, "k"), 1.0)
        P.api.gen_fill(v_in[i], c.req.seed, W.cache_stream(i, "v"), 1.0)
    return mw, k_in, v_in, to_dev(c.tok, torch.int32), to_dev(c.pos, torch.int32)


def force_tensor(S, L, N):
    fs = np.full((L, N), -1, dtype=np.int32)
    for i in range(1, L):
        fs[i, :len(S[i])] = S[i]
    return to_dev(fs, torch.int32)


def run_gpu(P, ctx, mw, k_in, v_in, tok, pos, c: Case, ks, force: bool):
    L, N = mw.shape.n_layers, c.N
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    sel = torch.full((L, N), -1, dtype=torch.int32, device=DEV)
    dev = torch.full((L, N), -1.0, dtype=torch.float32, device=DEV)
    fs = force_tensor(c.S, L, N) if force else None
    h = P.blend_forward(ctx, mw, tok, pos, list(c.cs), 0, k_in, v_in, kb, vb, ks, force_sel=fs, sel_out=sel,
                        dev_out=dev)
    torch.cuda.synchronize()
    ctx.check_device_errors()
    sels = [r[r >= 0] for r in sel.cpu().numpy()]
    return dict(kb=kb, vb=vb, sel=sels, dev=dev.cpu().numpy(), h=h.float().cpu().numpy())


# ---- comparisons (each returns a list of failure strings; empty = pass) -----------------------------------
def _f32(t):
    return t.float().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t, np.float32)


def row_head_errors(g: np.ndarray, o: np.ndarray) -> np.ndarray:
    """Relative L2 error per (row, kv head) of [R][H][hd] arrays."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    num = np.linalg.norm(g - o, axis=-1)
    den = np.maximum(np.linalg.norm(o, axis=-1), 1e-30)
    return num / den


def check_kv(kb, vb, Kc, Vc, ora, S, L, stats, tag="") -> List[str]:
    bad = []
    for i in range(L):
        kg, vg = _f32(kb[i]), _f32(vb[i])
        ko, vo = ora["K"][i], ora["V"][i]
        fresh = S[i] if i > 0 else np.zeros(0, np.int64)
        if len(fresh):
            ek = row_head_errors(kg[fresh], ko[fresh])
            ev = row_head_errors(vg[fresh], vo[fresh])
            stats[f"{tag}K{i}_fresh_max"] = float(ek.max())
            stats[f"{tag}V{i}_fresh_max"] = float(ev.max())
            if ek.max() > KV_TOL:
                r, h = np.unravel_index(ek.argmax(), ek.shape)
                bad.append(f"{tag}layer {i}: fresh K row {fresh[r]} head {h} rel err {ek.max():.3e} > {KV_TOL}")
            if ev.max() > KV_TOL:
                r, h = np.unravel_index(ev.argmax(), ev.shape)
                bad.append(f"{tag}layer {i}: fresh V row {fresh[r]} head {h} rel err {ev.max():.3e} > {KV_TOL}")
        keep = np.setdiff1d(np.arange(kg.shape[0]), fresh)
        if len(keep):
            if not np.array_equal(vg[keep], np.asarray(Vc[i], np.float32)[keep]):
                bad.append(f"{tag}layer {i}: untouched V rows are not the cache bytes")
            d = np.abs(kg[keep].astype(np.float64) - ko[keep])
            rowmax = np.abs(ko[keep]).reshape(len(keep), -1).max(axis=1)[:, None, None]
            lim = 2.0 ** -8 * np.abs(ko[keep]) + 1e-5 * rowmax
            stats[f"{tag}K{i}_untouched_ratio"] = float((d / lim).max())
            if np.any(d > lim):
                bad.append(f"{tag}layer {i}: untouched K exceeds the bf16 realign bound ({(d / lim).max():.2f}x)")
    return bad


def check_dev(dev_gpu, ora, S, L, stats, tag="") -> List[str]:
    """dev_gpu: [L][N] in candidate order (C_1 = all tokens, C_i = S_{i-1})."""
    bad = []
    for i in range(1, L):
        rows, do = ora["dev"][i]
        cand = S[i - 1]
        dg = np.asarray(dev_gpu[i][:len(cand)], np.float64)[np.searchsorted(cand, rows)]
        err = np.abs(dg - do) / np.maximum(do, 1e-30)
        stats[f"{tag}dev{i}_max_rel"] = float(err.max())
        if err.max() > DEV_TOL:
            j = err.argmax()
            bad.append(f"{tag}layer {i}: Delta_kv of token {rows[j]}: gpu {dg[j]:.6g} oracle {do[j]:.6g}")
    return bad


def check_h(h_gpu, ora, S_last, stats, tag="") -> List[str]:
    idx = np.searchsorted(S_last, ora["h_rows"])
    g = np.asarray(h_gpu, np.float64)[idx]
    o = ora["h"]
    e = np.linalg.norm(g - o, axis=1) / np.maximum(np.linalg.norm(o, axis=1), 1e-30)
    stats[f"{tag}h_max_rel"] = float(e.max())
    if e.max() > H_TOL:
        return [f"{tag}final h row {ora['h_rows'][e.argmax()]}: rel err {e.max():.3e} > {H_TOL}"]
    return []


def check_free_selection(sel, dev_gpu, ora, ks, N, stats, tag="") -> List[str]:
    """Free-running selections: sorted, sized, nested, the exact top-k of the GPU's own Delta_kv (ties -> lower
    token, R6); S_1 equal to the oracle's top-k_1 (over all N tokens) except flips inside the measured Delta_kv
    error band (tests.helpers.band_check)."""
    bad = []
    prev = np.arange(N)
    for i in range(1, len(ks)):
        si = sel[i]
        if len(si) != ks[i] or np.any(np.diff(si) <= 0) or not np.isin(si, prev).all():
            bad.append(f"{tag}layer {i}: S_i not sorted / sized / nested")
        if not np.array_equal(topk_tokens(dev_gpu[i][:len(prev)], prev, ks[i]), si):
            bad.append(f"{tag}layer {i}: S_i is not the top-k of the reported Delta_kv")
        prev = si
    rows, do = ora["dev"][1]
    assert np.array_equal(rows, np.arange(N))
    dg = np.asarray(dev_gpu[1][:N], np.float64)
    ok, flips, band = band_check(sel[1], dg, do, rows, ks[1])
    stats[f"{tag}S1_flips"] = flips
    stats[f"{tag}S1_band"] = band
    if not ok:
        bad.append(f"{tag}layer 1: {flips} selection flips, some outside the measured Delta_kv error band {band:.3g}")
    return bad
