"""Interleaved A/B timing of the Mistral 6x512 blend under two option sets (one CUDA graph each, replayed
alternately so clock / power drift hits both equally).
python tools/ab.py "gemm_no192=1" "gemm_no192=0" [rounds] [--e2e]
--e2e: the request path (cb_blend_request: pinned host chunk KV, layer-pipelined H2D, h_out D2H) instead of
the device-resident forward."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def opts(spec):
    return [(k, int(v)) for k, v in (kv.split("=") for kv in spec.split(",") if kv)]


def main():
    e2e = "--e2e" in sys.argv
    argv = [a for a in sys.argv if a != "--e2e"]
    A, B = argv[1], argv[2]
    rounds = int(argv[3]) if len(argv) > 3 else 40
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    req = W.Request([512] * 6, 0, 1, 0.15)
    N, L = req.n_ctx, s.n_layers
    dev = torch.device("cuda", 0)
    mw = P.ModelWeights.synth(s, 1, "bf16", dev)
    tok = torch.from_numpy(req.tokens(s.vocab)).to(dev)
    pos = torch.from_numpy(req.global_positions()).to(dev)
    cs = req.chunk_starts()
    k_in = torch.randn(L, N, s.n_kv_heads, s.head_dim, device=dev).to(torch.bfloat16)
    v_in = torch.randn_like(k_in)
    ks = P.schedule(0.15, N, L)
    graphs = {}
    for name, spec in (("A", A), ("B", B)):
        # a context of its own per option set: options set for A must not leak into B's graph
        ctx = P.Context(s, "bf16", max_tokens=N, max_pos=2 * N)
        for k, v in opts(spec):
            ctx.set_option(k, v)
        kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
        h_out = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=dev)
        f = lambda kb=kb, vb=vb, h_out=h_out, ctx=ctx: P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, kb, vb, ks,
                                                               h_out=h_out)
        if e2e:
            kh, vh = k_in.cpu().pin_memory(), v_in.cpu().pin_memory()
            toks, poss = tok.cpu().pin_memory(), pos.cpu().pin_memory()
            hh = torch.empty(ks[-1], s.d_model, dtype=torch.float32).pin_memory()
            f = lambda kb=kb, vb=vb, kh=kh, vh=vh, toks=toks, poss=poss, hh=hh, ctx=ctx: P.api.blend_request(
                ctx, mw, toks, poss, list(cs), 0, kh, vh, kb, vb, ks, hh)
        f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[name] = (g, f, kb, vb, h_out, ctx)
    for _ in range(3):
        for g, *_ in graphs.values():
            g.replay()
    torch.cuda.synchronize()
    times = {"A": [], "B": []}
    for r in range(rounds):
        for name in (("A", "B") if r % 2 == 0 else ("B", "A")):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graphs[name][0].replay()
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1))
    for name, spec in (("A", A), ("B", B)):
        t = times[name]
        print(f"{name} [{spec}]: median {statistics.median(t):.3f} ms  mean {np.mean(t):.3f} +- {np.std(t):.3f}")
    d = np.array(times["A"]) - np.array(times["B"])
    print(f"A - B: mean {d.mean():.3f} ms, median {np.median(d):.3f} ms (paired)")


if __name__ == "__main__":
    main()
