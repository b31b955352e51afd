"""Full-depth parity of the bench workload against the fp64 oracle: the Mistral-7B-shape 6x512 request at
r = 0.15 through all 32 layers, in replay mode (R14: the seeded nested selections forced on both sides), the
GPU blend in the bench's launch configuration against `oracle.blend_replay_rows` over every row the outputs
depend on. Prints, per layer, the largest per-(row, kv head) relative L2 error of the fresh K / V rows (S_i),
the untouched-K bound ratio, whether untouched V rows are the cache bytes, the largest relative Delta_kv error
over the layer's candidates, and the final h rows' largest per-row relative L2 error.

python tools/full_depth_parity.py [model] [ratio]   (needs a B200; the oracle takes ~1-2 min on 16 host threads)
Test infrastructure: reads the oracle, like tests/; the numbers go to DESIGN.md §3."""
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "mistral-7b"
    ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from oracle import cacheblend_oracle as O
    from synth import workload as W
    from tests import fullsize as F
    full = W.MODELS[model]
    lens = {"mistral-7b": [512] * 6, "yi-34b": [1024] * 8, "llama-70b": [1024] * 10}[model]
    rs = F.SEED
    req = W.Request(list(lens), 0, rs, ratio)
    N, L = req.n_ctx, full.n_layers
    ks = O.schedule(ratio, N, L)
    S = W.nested_selection(rs, N, ks)
    Kc = np.stack([W.random_cache(full, i, N, rs, "bf16", "k") for i in range(L)])
    Vc = np.stack([W.random_cache(full, i, N, rs, "bf16", "v") for i in range(L)])
    c = F.Case(f"{model}-full", full, full, req, F.SEED, req.tokens(full.vocab), req.global_positions(),
               req.chunk_starts(), ks, ks, S, S[-1], Kc, Vc)
    # GPU first (frees its memory before the oracle's fp64 arrays grow)
    mw, k_in, v_in, tok, pos = F.gpu_inputs(P, c, shape=full)
    ctx = P.Context(full, "bf16", max_tokens=N, max_pos=2 * N)
    g = F.run_gpu(P, ctx, mw, k_in, v_in, tok, pos, c, ks, force=True)
    kb = g["kb"].float().cpu().numpy()
    vb = g["vb"].float().cpu().numpy()
    dev_gpu, h_gpu = g["dev"], g["h"]
    del mw, k_in, v_in, ctx, g
    torch.cuda.empty_cache()
    t = time.time()
    emb = W.embed_weights(full, F.SEED, "bf16")[c.tok]
    ora = O.blend_replay_rows(c.tok, c.pos, c.cs, Kc, Vc, S, F.layer_model(full, F.SEED), emb,
                              dev_rows_1=np.arange(N), h_rows_last=S[-1], threads=F.THREADS)
    t_ora = time.time() - t
    rows = []
    for i in range(L):
        fresh = S[i] if i > 0 else np.zeros(0, np.int64)
        r = {"layer": i}
        if len(fresh):
            r["K_fresh_max"] = float(F.row_head_errors(kb[i][fresh], ora["K"][i][fresh]).max())
            r["V_fresh_max"] = float(F.row_head_errors(vb[i][fresh], ora["V"][i][fresh]).max())
        keep = np.setdiff1d(np.arange(N), fresh)
        d = np.abs(kb[i][keep].astype(np.float64) - ora["K"][i][keep])
        rowmax = np.abs(ora["K"][i][keep]).reshape(len(keep), -1).max(axis=1)[:, None, None]
        r["K_untouched_ratio"] = float((d / (2.0 ** -8 * np.abs(ora["K"][i][keep]) + 1e-5 * rowmax)).max())
        r["V_untouched_bitwise"] = bool(np.array_equal(vb[i][keep], np.asarray(Vc[i], np.float32)[keep]))
        if i >= 1:
            drows, do = ora["dev"][i]
            cand = S[i - 1]
            dg = np.asarray(dev_gpu[i][:len(cand)], np.float64)[np.searchsorted(cand, drows)]
            r["dev_max_rel"] = float((np.abs(dg - do) / np.maximum(do, 1e-30)).max())
        rows.append(r)
    idx = np.searchsorted(S[-1], ora["h_rows"])
    hg = np.asarray(h_gpu, np.float64)[idx]
    eh = np.linalg.norm(hg - ora["h"], axis=1) / np.maximum(np.linalg.norm(ora["h"], axis=1), 1e-30)
    print(f"model {model} {len(lens)}x{lens[0]} r={ratio}: oracle {t_ora:.1f} s on {F.THREADS} threads")
    print("layer  K_fresh_max  V_fresh_max  K_untouched_ratio  V_bitwise  dev_max_rel")
    for r in rows:
        print(f"{r['layer']:5d}  {r.get('K_fresh_max', float('nan')):11.3e}  {r.get('V_fresh_max', float('nan')):11.3e}"
              f"  {r['K_untouched_ratio']:17.3f}  {str(r['V_untouched_bitwise']):>9s}  {r.get('dev_max_rel', float('nan')):11.3e}")
    print(f"final h ({len(eh)} rows): max rel L2 {eh.max():.3e}, median {np.median(eh):.3e}")
    print(json.dumps({"model": model, "ratio": ratio, "layers": rows, "h_max_rel": float(eh.max()),
                      "h_median_rel": float(np.median(eh)), "oracle_s": t_ora}))


if __name__ == "__main__":
    main()
