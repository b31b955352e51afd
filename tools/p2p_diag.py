"""Loopback diagnostics of the peer-memory collectives: two tiny fp32 head-parallel ranks on one GPU, forward
in two threads, flag words of both ranks printed while / after it runs.  python tools/p2p_diag.py [p2p 0|1]"""
import ctypes
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p2p = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    import paper_2405_16444_b200 as P
    from paper_2405_16444_b200 import dist as D
    from synth import workload as W
    import dataclasses
    name = sys.argv[3] if len(sys.argv) > 3 else "tiny"
    dt = "f32" if name == "tiny" else "bf16"
    s = dataclasses.replace(W.MODELS[name], n_layers=3) if name == "tiny" else W.MODELS[name]
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    req = W.Request([32, 32, 32] if name == "tiny" else [512] * 6, 0, 1, 0.2)
    N = req.n_ctx
    ss = D.head_shard_shape(s, world)
    g = P.Group(world)
    full = P.ModelWeights.synth(s, 1, dt, "cuda")
    tok = torch.from_numpy(req.tokens(s.vocab)).cuda()
    pos = torch.from_numpy(req.global_positions()).cuda()
    ks = P.schedule(0.2, N, s.n_layers)
    ranks = []
    for r in range(world):
        ctx = P.Context(ss, dt, max_tokens=N, max_pos=2 * N)
        for kv in filter(None, os.environ.get("CB_OPTS", "").split(",")):  # e.g. CB_OPTS=gemm_pair=2
            k_, v_ = kv.split("=")
            ctx.set_option(k_, int(v_))
        ctx.set_comm_local(g, r)
        if p2p:
            if p2p == 2:
                ctx.set_option("tp_fuse", 0)
            ctx.enable_tp_p2p()
        mw = P.ModelWeights(ss, dt, full.embed, [D.shard_layer(w, s, r, world) for w in full.layers])
        k = torch.randn(s.n_layers, N, ss.n_kv_heads, s.head_dim, device="cuda").to(P.api.TORCH_DTYPES[dt])
        ranks.append(dict(ctx=ctx, mw=mw, k=k, v=torch.randn_like(k), kb=torch.empty_like(k), vb=torch.empty_like(k),
                          h=torch.empty(ks[-1], s.d_model, device="cuda"), st=torch.cuda.Stream()))
    torch.cuda.synchronize()
    t0 = time.time()
    done = [None] * world

    def work(r):
        x = ranks[r]
        P.blend_forward(x["ctx"], x["mw"], tok, pos, list(req.chunk_starts()), 0, x["k"], x["v"], x["kb"], x["vb"], ks,
                        h_out=x["h"], stream=x["st"])
        done[r] = ("enqueued", time.time() - t0)
        x["st"].synchronize()
        done[r] = ("finished", time.time() - t0)

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    if os.environ.get("CB_DIAG_NOPOLL"):  # no flag reads while it runs: only the per-rank finish times
        for t in th:
            t.join(timeout=60)
        print("nopoll", done, flush=True)
        os._exit(0)
    for it in range(12):
        time.sleep(2)
        line = [f"t={time.time() - t0:.0f}s"]
        tags = []
        for r, x in enumerate(ranks):
            if p2p:
                fb = torch.zeros(53, dtype=torch.int32).pin_memory()
                P.api.check(P.api.lib().cb_debug_p2p_flags(x["ctx"].handle,
                                                           ctypes.cast(fb.data_ptr(), ctypes.POINTER(ctypes.c_int32))))
                f = fb.tolist()
                ring = [tuple(f[20 + 4 * i:24 + 4 * i]) for i in range(8)]
                tags.append(f[52])
                ring = [(q, (rkm % 256) // 16, rkm % 16, f"wait {rkm // 256} us") for q, rkm, b0, b1 in ring if q]
                line.append(f"r{r} {done[r]} entry {list(f[:world])} exit {list(f[8:8 + world])} seq {f[16]} "
                            f"cnt {f[17]} ring {sorted(ring)}")
            else:
                line.append(f"r{r} {done[r]}")
        print(" | ".join(line), [hex(t & 0xffffff) for t in tags], flush=True)
        if all(d and d[0] == "finished" for d in done):
            break
    print("launches", [x["ctx"].launch_count() for x in ranks], flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
