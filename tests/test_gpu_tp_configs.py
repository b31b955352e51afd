"""Head-parallel blend (SURVEY.md §8(e) partitioning 1) at the BASELINE configurations' full width, on one GPU
through the loopback group (each rank a context of the shard model driven by its own host thread and stream,
the same per-rank kernels the NCCL path runs; tests/test_gpu_tp.py covers the group mechanics and NCCL):

- Mistral-7B 6x512 over 2 ranks (16/4 heads, d_ff 7168 per rank);
- Yi-34B 8x1024 over 8 ranks (the TP8 shard: 7 q heads / 1 kv head, GQA 7, d_ff 2560) and over 4 (14/2);
- Llama-70B 10x1024 over 8 ranks (the TP8 shard: 8 q / 1 kv head, d_ff 3584).

Each against the SAME fp64 oracle replay as the single-GPU test (tests/fullsize.py: truncated depth, seeded
inputs and forced selections, per-(row, head) / per-row tolerances): K/V reassembled over the ranks' kv heads,
Delta_kv, the final h rows, and the free-running S_1 against the oracle's own top-k inside the measured error
band. Every rank must hold bitwise the same S_i, Delta_kv and h (one top-k over the gathered partials)."""
import threading

import numpy as np
import pytest
import torch

from paper_2405_16444_b200 import dist as D
from tests import fullsize as F

pytestmark = pytest.mark.gpu


def _forward_tp(P, c, mw_full, world, k_in, v_in, tok, pos, force: bool):
    s = c.s
    ss = D.head_shard_shape(s, world)
    g = P.Group(world)
    L, N = s.n_layers, c.N
    fs = F.force_tensor(c.S, L, N) if force else None
    ranks = []
    for r in range(world):
        ctx = P.Context(ss, "bf16", max_tokens=N, max_pos=2 * N)
        ctx.set_comm_local(g, r)
        mw = P.ModelWeights(ss, "bf16", mw_full.embed, [D.shard_layer(w, s, r, world) for w in mw_full.layers])
        ki, vi = D.shard_kv(k_in, s, r, world), D.shard_kv(v_in, s, r, world)
        ranks.append(dict(ctx=ctx, mw=mw, ki=ki, vi=vi, kb=torch.empty_like(ki), vb=torch.empty_like(vi),
                          sel=torch.full((L, N), -1, dtype=torch.int32, device=F.DEV),
                          dev=torch.full((L, N), -1.0, dtype=torch.float32, device=F.DEV),
                          h=torch.empty(c.ks[-1], s.d_model, dtype=torch.float32, device=F.DEV),
                          st=torch.cuda.Stream()))
    torch.cuda.synchronize()
    errs = [None] * world

    def work(r):
        x = ranks[r]
        try:
            P.blend_forward(x["ctx"], x["mw"], tok, pos, list(c.cs), 0, x["ki"], x["vi"], x["kb"], x["vb"], c.ks,
                            force_sel=fs, sel_out=x["sel"], dev_out=x["dev"], h_out=x["h"], stream=x["st"])
            x["st"].synchronize()
        except Exception as e:  # surfaced below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(not t.is_alive() for t in th), "a rank hung"
    for e in errs:
        if e is not None:
            raise e
    for x in ranks:
        x["ctx"].check_device_errors()
    for x in ranks[1:]:  # every rank took the same decisions on the same numbers
        assert torch.equal(x["sel"], ranks[0]["sel"])
        assert torch.equal(x["dev"], ranks[0]["dev"])
        assert torch.equal(x["h"], ranks[0]["h"])
    sel = [r_[r_ >= 0] for r_ in ranks[0]["sel"].cpu().numpy()]
    return dict(kb=torch.cat([x["kb"] for x in ranks], dim=2), vb=torch.cat([x["vb"] for x in ranks], dim=2),
                sel=sel, dev=ranks[0]["dev"].cpu().numpy(), h=ranks[0]["h"].cpu().numpy())


@pytest.mark.parametrize("name,world", [("mistral15", 2), ("yi15", 8), ("yi15", 4), ("llama15", 8)])
def test_tp_config_parity(P, name, world):
    c = F.case_for(name)
    ora = F.oracle(c)
    mw, k_in, v_in, tok, pos = F.gpu_inputs(P, c)
    stats, bad = {}, []
    rep = _forward_tp(P, c, mw, world, k_in, v_in, tok, pos, force=True)
    for i in range(1, F.L_T):
        if not np.array_equal(rep["sel"][i], c.S[i]):
            bad.append(f"layer {i}: replay did not keep the forced selection")
    bad += F.check_kv(rep["kb"], rep["vb"], c.Kc, c.Vc, ora, c.S, F.L_T, stats)
    bad += F.check_dev(rep["dev"], ora, c.S, F.L_T, stats)
    bad += F.check_h(rep["h"], ora, c.S[-1], stats)
    free = _forward_tp(P, c, mw, world, k_in, v_in, tok, pos, force=False)
    bad += F.check_free_selection(free["sel"], free["dev"], ora, c.ks, c.N, stats)
    print(name, world, {k: (round(v, 5) if isinstance(v, float) else v) for k, v in stats.items()})
    assert not bad, "\n".join(bad)
