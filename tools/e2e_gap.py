"""Where the request path's end-to-end time goes: interleaved replays (one CUDA graph each) of
  dev  -- cb_blend_forward on device-resident chunk KV (the bench's device-timed step),
  req  -- cb_blend_request from pinned host chunk KV (layer-pipelined H2D on the copy stream, h_out D2H),
  reqd -- cb_blend_request with the chunk KV already in device memory (the same copies become D2D),
on the Mistral 6x512 bench workload. python tools/e2e_gap.py [rounds]   (needs a B200)"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    req = W.Request([512] * 6, 0, 1, 0.15)
    N, L = req.n_ctx, s.n_layers
    dev = torch.device("cuda", 0)
    ctx = P.Context(s, "bf16", max_tokens=N, max_pos=2 * N)
    mw = P.ModelWeights.synth(s, 1, "bf16", dev)
    tok = torch.from_numpy(req.tokens(s.vocab)).to(dev)
    pos = torch.from_numpy(req.global_positions()).to(dev)
    cs = list(req.chunk_starts())
    k_in = torch.randn(L, N, s.n_kv_heads, s.head_dim, device=dev).to(torch.bfloat16)
    v_in = torch.randn_like(k_in)
    ks = P.schedule(0.15, N, L)
    kh, vh = k_in.cpu().pin_memory(), v_in.cpu().pin_memory()
    toks, poss = tok.cpu().pin_memory(), pos.cpu().pin_memory()
    fns = {}
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    h_out = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=dev)
    hh = torch.empty(ks[-1], s.d_model, dtype=torch.float32).pin_memory()
    fns["dev"] = lambda: P.blend_forward(ctx, mw, tok, pos, cs, 0, k_in, v_in, kb, vb, ks, h_out=h_out)
    fns["req"] = lambda: P.api.blend_request(ctx, mw, toks, poss, cs, 0, kh, vh, kb, vb, ks, hh)
    fns["reqd"] = lambda: P.api.blend_request(ctx, mw, toks, poss, cs, 0, k_in, v_in, kb, vb, ks, hh)
    graphs = {}
    for name, f in fns.items():
        f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[name] = g
    for _ in range(3):
        for g in graphs.values():
            g.replay()
    torch.cuda.synchronize()
    times = {k: [] for k in graphs}
    names = list(graphs)
    for r in range(rounds):
        order = names if r % 2 == 0 else names[::-1]
        for name in order:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graphs[name].replay()
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1))
    for name in names:
        t = times[name]
        print(f"{name:5s}: median {statistics.median(t):.3f} ms  mean {np.mean(t):.3f} +- {np.std(t):.3f}")
    for a, b in (("req", "dev"), ("reqd", "dev"), ("req", "reqd")):
        d = np.array(times[a]) - np.array(times[b])
        print(f"{a} - {b}: median {np.median(d):.3f} ms (paired)")


if __name__ == "__main__":
    main()
