#!/usr/bin/env python
"""Benchmark: CacheBlend blend_forward at 15 % recompute, Mistral-7B shape, 6 x 512-token chunks
(BASELINE.json metric / configs[1]) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config mistral]

One step = one cb_blend_forward over one request (realign + layer 0 + 31 selective layers), inputs
resident in HBM. Multi-GPU (torchrun, N>1): request-parallel, each rank blends its own request
(weak scaling, no collective on the data path; SURVEY §8(e) partitioning 2). Prints ONE JSON line
on rank 0. --impl reference times the fp64 CPU oracle (bounded sample) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import workload as W  # noqa: E402

CONFIGS = {  # name -> (model shape, chunk lens, ratio)
    "mistral": ("mistral-7b", [512] * 6, 0.15),
    "yi": ("yi-34b", [1024] * 8, 0.15),
    "llama": ("llama-70b", [1024] * 10, 0.15),
    "small": ("small", [200, 317, 150], 0.15),
}
METRIC = "blend latency ms & context tok/s at 15% recompute (Mistral-7B shape)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mistral", choices=sorted(CONFIGS) + ["batched"],
                    help="batched = SURVEY config 5: 64 Mistral-shape requests of 4-8 chunks x 256-1024 "
                         "tokens, assigned to the ranks longest-first")
    ap.add_argument("--batched-requests", type=int, default=64)
    ap.add_argument("--tp-comm", default="nccl", choices=["nccl", "p2p"],
                    help="--parallel heads: NCCL calls (default) or the library's NVLink peer-memory collectives "
                         "(o_proj / down_proj epilogues push rows to their owners; experimental, DESIGN.md §7)")
    ap.add_argument("--parallel", default="auto", choices=["auto", "request", "heads"],
                    help="N>1: head-parallel tensor parallelism over the N GPUs (strong scaling, NCCL all-gather / "
                         "all-reduces inside the blend; the default, BASELINE north_star 'head-partitioned at 2, 4 "
                         "and 8 GPUs') with a request-parallel sub-record (weak scaling, no collective), or "
                         "request-parallel only")
    ap.add_argument("--ratio", type=float, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--attn-deviation", action="store_true", help="GPU measurement of the attention deviation "
                    "curve (SURVEY §8(f) N2, Fig. ca_reduction) for --config, then exit")
    ap.add_argument("--cpu-full", action="store_true", help="time one whole fp64 oracle blend (layer-streamed "
                    "weights) and the sampled estimate, then exit (validates the cpu_baseline extrapolation)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-request-sub", action="store_true", help="N>1 head-parallel: skip the request-parallel "
                    "sub-record")
    ap.add_argument("--no-baselines", action="store_true", help="skip the full-prefill / full-reuse timings")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of one CUDA graph per step")
    ap.add_argument("--no-pdl", action="store_true", help="disable programmatic dependent launch")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------------
# algorithmic work; the avoided dense work is not counted
# ---------------------------------------------------------------------------------------------------
def algorithmic_work(s, N, n_suf, ks, sel=None):
    """SURVEY §8(d) algorithmic FLOPs and bytes of one blend, per kernel class.

    sel: the step's selected token ids per layer (sel[0] unused, layer 0 is full). Attention is then
    counted exactly, 4 qd (g_j + 1) FLOP per query j with global position g_j = j (positions 0..T-1);
    without it, with the mean causal span of the kept queries estimated as (T + 1) / 2."""
    d, qd, kvd, ff, L = s.d_model, s.qd, s.kvd, s.d_ff, s.n_layers
    T = N + n_suf
    B = 2
    g = np.arange(T, dtype=np.float64)  # positions 0..T-1: causal span of token t is t + 1
    tot_gemm = 2.0 * T * (d * qd + qd * d + 3 * d * ff) + 2.0 * n_suf * d * 2 * kvd
    attn = 4.0 * qd * float(np.sum(g + 1))
    dev_bytes = topk_bytes = scatter_bytes = 0.0
    cand = N
    exact = sel is not None
    for i in range(1, L):
        k = ks[i]
        tot_gemm += 2.0 * (cand + n_suf) * d * (qd + 2 * kvd) + 2.0 * (k + n_suf) * (qd * d + 3 * d * ff)
        if exact:
            span = float(np.sum(np.asarray(sel[i], dtype=np.float64) + 1)) + float(np.sum(g[N:] + 1))
        else:
            span = (k + n_suf) * (T + 1) / 2.0
        attn += 4.0 * qd * span
        dev_bytes += cand * 2 * kvd * B                      # cached K^, V rows of the candidates (fused)
        topk_bytes += cand * (2 * ((kvd + 63) // 64)) * 4    # per-block Delta_kv partials, fp32
        scatter_bytes += (k + n_suf) * 2 * kvd * B * 2       # fresh rows read + written into the cache
        cand = k
    wbytes = L * B * (d * qd + 2 * d * kvd + qd * d + 3 * d * ff)
    realign_k = 2.0 * L * N * kvd * B            # K read + write (the algorithmic work)
    realign_bytes = 2.0 * realign_k              # out of place: V carried over too (read + write)
    attn_bytes = L * T * 2 * kvd * B             # every layer's blended K/V read once
    return dict(gemm_flops=tot_gemm, attn_flops=attn, attn_exact=float(exact), weight_bytes=wbytes,
                realign_bytes=realign_bytes, realign_k_bytes=realign_k, attn_bytes=attn_bytes,
                dev_bytes=dev_bytes, topk_bytes=topk_bytes, scatter_bytes=scatter_bytes)


def path_roofline(work, prof, ms_step, hbm, tf):
    """Whole-path fraction: sum over kernel classes of max(FLOP / tensor peak, bytes / HBM
    peak), divided by the measured step time. prof: measured ms per class (per-launch CUDA events)."""
    ideal = {
        "gemm": max(work["gemm_flops"] / (tf * 1e9), work["weight_bytes"] / (hbm * 1e6)),
        "attention": max(work["attn_flops"] / (tf * 1e9), work["attn_bytes"] / (hbm * 1e6)),
        "realign": work["realign_k_bytes"] / (hbm * 1e6),
        "topk": work["topk_bytes"] / (hbm * 1e6),
        "scatter": work["scatter_bytes"] / (hbm * 1e6),
    }
    tot = sum(ideal.values())
    per = {k: {"ideal_ms": round(v, 4), "ms": round(prof.get(k, 0.0), 4),
               "frac": round(v / prof[k], 3) if prof.get(k) else None} for k, v in ideal.items()}
    return {"frac": tot / ms_step, "ideal_ms": tot, "ms_per_step": ms_step, "per_class": per,
            "note": "sum of per-class max(FLOP/tensor peak, bytes/HBM peak) over the measured step time; "
                    "GEMM and attention FLOPs on the tensor peak, realign (K read+write only), top-k partials "
                    "and scatter on HBM; the deviation is fused into the QKV epilogue (inside gemm)"}


# ---------------------------------------------------------------------------------------------------
# clocks sampled DURING the timed region
# ---------------------------------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j["hbm_gbs"], j["bf16_tflops"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference): bounded sample of the same workload
# ---------------------------------------------------------------------------------------------------
class OracleSample:
    """Realign of every layer + layers 0, 1, 2 of the blend, run by the fp64 oracle as it stands, on the
    same shapes (random-cache mode inputs: values do not change the oracle's cost). Later layers are
    extrapolated from layer 2 in proportion to their candidate/kept row counts."""

    def __init__(self, s, lens, ratio, seed):
        from oracle import cacheblend_oracle as O
        self.O, self.s = O, s
        self.req = W.Request(list(lens), 0, seed, ratio)
        N = self.req.n_ctx
        self.ks = O.schedule(ratio, N, s.n_layers)
        n_layers = min(3, s.n_layers)
        self.model = O.Model.build(s, W.embed_weights(s, seed, "bf16"),
                                   [W.layer_weights(s, i, seed, "bf16") for i in range(n_layers)])
        self.tok, self.pos = self.req.tokens(s.vocab), self.req.global_positions()
        self.loc = self.req.local_positions()
        self.Kc = W.random_cache(s, 0, N, seed, "bf16", "k").astype(np.float64)
        self.Vc = W.random_cache(s, 0, N, seed, "bf16", "v").astype(np.float64)

    def run(self):
        O, s, m = self.O, self.s, self.model
        N, L = self.req.n_ctx, s.n_layers
        t0 = time.perf_counter()
        K = np.zeros((3, N, s.n_kv_heads, s.head_dim))
        V = np.zeros_like(K)
        for i in range(L):  # realign every layer (the oracle's step 1)
            Ki = O.realign(self.Kc, self.loc, self.pos, s.rope_theta)
            if i < 3:
                K[i], V[i] = Ki, self.Vc
        t_realign = time.perf_counter() - t0
        t1 = time.perf_counter()
        h = m.embed[self.tok]
        q, _, _ = O.qkv(m, 0, h, self.pos)
        a = O.causal_attention(q, self.pos, K[0], V[0], self.pos)
        h = O.attn_out_mlp(m, 0, h, a)
        t_l0 = time.perf_counter() - t1
        cand = np.arange(N)
        t_layers = []
        for i in (1, 2):
            t2 = time.perf_counter()
            h, sel, _ = O.blend_layer(m, i, h, cand, N, 0, self.ks[i], K, V, self.pos)
            t_layers.append(time.perf_counter() - t2)
            cand = sel
        # layers 3..L-1 ~ layer 2 scaled by rows (candidates for QKV, kept rows for the rest)
        w2 = self.ks[1] + self.ks[2]
        rest = sum(self.ks[i - 1] + self.ks[i] for i in range(3, L)) / w2 * t_layers[1]
        total = t_realign + t_l0 + sum(t_layers) + rest
        sample = time.perf_counter() - t0
        return total, sample

    @staticmethod
    def cores():
        try:
            from threadpoolctl import threadpool_info
            return max(int(x.get("num_threads", 1)) for x in threadpool_info()) or os.cpu_count()
        except Exception:
            return os.cpu_count()


class _StreamedLayers:
    """The oracle Model's layer list with layer-streamed weights: layer i is generated (synth recipe, the
    oracle's own input path) when first indexed and replaced by the next layer, so one layer's fp64
    weights are resident at a time. gen_s accumulates the (untimed) generation time."""

    def __init__(self, s, seed):
        self.s, self.seed, self.i, self.w, self.gen_s = s, seed, -1, None, 0.0

    def __len__(self):
        return self.s.n_layers

    def __getitem__(self, i):
        if i != self.i:
            t = time.perf_counter()
            self.w = None
            self.w = {k: np.asarray(v, dtype=np.float64) for k, v in W.layer_weights(self.s, i, self.seed,
                                                                                   "bf16").items()}
            self.i = i
            self.gen_s += time.perf_counter() - t
        return self.w


def oracle_full_blend(s, lens, ratio, seed):
    """The whole fp64 oracle blend of one request (realign + layer 0 + layers 1..L-1), layer-streamed
    weights, random chunk caches. Returns (compute seconds excluding weight generation, generation s)."""
    from oracle import cacheblend_oracle as O
    req = W.Request(list(lens), 0, seed, ratio)
    N, L = req.n_ctx, s.n_layers
    ks = O.schedule(ratio, N, L)
    layers = _StreamedLayers(s, seed)
    m = O.Model(L, s.d_model, s.n_q_heads, s.n_kv_heads, s.head_dim, s.rope_theta, s.rms_eps,
                np.asarray(W.embed_weights(s, seed, "bf16"), dtype=np.float64), layers)
    tok, pos, loc = req.tokens(s.vocab), req.global_positions(), req.local_positions()
    Kc = np.stack([W.random_cache(s, i, N, seed, "bf16", "k") for i in range(L)]).astype(np.float64)
    Vc = np.stack([W.random_cache(s, i, N, seed, "bf16", "v") for i in range(L)]).astype(np.float64)
    layers[0]
    g0 = layers.gen_s
    t0 = time.perf_counter()
    res = O.blend_forward(m, tok, pos, req.chunk_starts(), 0, Kc, Vc, ks)
    wall = time.perf_counter() - t0
    return wall - (layers.gen_s - g0), layers.gen_s, res


def run_cpu_full(args):
    """One full oracle blend of the bench workload (validates the sampled cpu_baseline's extrapolation)."""
    shape_name, lens, ratio = CONFIGS.get(args.config, CONFIGS["mistral"])
    s = W.MODELS[shape_name]
    smp = OracleSample(s, lens, ratio, args.seed)
    est, sample_s = smp.run()
    full_s, gen_s, _ = oracle_full_blend(s, lens, ratio if args.ratio is None else args.ratio, args.seed)
    N = sum(lens)
    print(json.dumps({"kind": "oracle full blend", "workload": f"{shape_name} {len(lens)}x{lens[0]} r={ratio}",
                      "full_blend_s": full_s, "full_ctx_tok_s": N / full_s, "weight_generation_s_untimed": gen_s,
                      "sampled_estimate_s": est, "sample_s": sample_s,
                      "estimate_over_full": est / full_s, "cores": OracleSample.cores()}), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    shape_name, lens, ratio = CONFIGS.get(args.config, CONFIGS["mistral"])  # batched: per-request Mistral
    ratio = args.ratio if args.ratio is not None else ratio
    s = W.MODELS[shape_name]
    smp = OracleSample(s, lens, ratio, args.seed)
    for _ in range(args.warmup):
        smp.run()
    est, samples = [], []
    for _ in range(args.steps):
        e, t = smp.run()
        est.append(e)
        samples.append(t)
    ms_blend = float(np.mean(est)) * 1e3      # one whole blend, extrapolated from the sample
    ms_step = float(np.mean(samples)) * 1e3   # what each step actually ran (the driver's clock sees this)
    N = sum(lens)
    v = N / (ms_blend / 1e3)
    cores = OracleSample.cores()
    sample = (f"per step: realign all {s.n_layers} layers + layers 0-2 in full (fp64 numpy, "
              f"{ms_step / 1e3:.1f} s measured); layers 3..{s.n_layers - 1} extrapolated from layer 2 by row counts "
              f"to {ms_blend / 1e3:.1f} s per blend (value = n_ctx / that); a full oracle blend timed once: "
              "profiles/r02_cpu_full_blend.json")
    line = {"metric": METRIC, "value": v, "unit": "ctx_tok/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_blend_extrapolated": ms_blend,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter RNG)", "impl": "reference",
            "config": {"workload": f"{shape_name} {len(lens)}x{lens[0]} tokens, r={ratio}, 1 request per GPU",
                       "recompute_ratio": ratio, "n_ctx": N, "parallelism": "request-parallel x1 (rank 0 only)"},
            "cpu_baseline": {"value": v, "unit": "ctx_tok/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "ctx_tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2405_16444_b200.build import build
    if rank == 0 or world == 1:
        build()
    if world > 1:
        dist.barrier()
    import paper_2405_16444_b200 as P

    shape_name, lens, ratio = CONFIGS[args.config]
    ratio = args.ratio if args.ratio is not None else ratio
    s = W.MODELS[shape_name]
    heads = args.parallel == "heads" or (args.parallel == "auto" and world > 1)
    # request-parallel (weak scaling): every rank blends its own request; head-parallel (strong scaling):
    # all ranks blend the same request, each with its heads / d_ff features
    seed = args.seed if heads else args.seed + rank
    req = W.Request(list(lens), 0, seed, ratio)
    N, L = req.n_ctx, s.n_layers
    dev = torch.device("cuda", local)
    from paper_2405_16444_b200 import dist as D
    sh = D.head_shard_shape(s, world) if heads else s  # the model this rank's context holds
    ctx = P.Context(sh, "bf16", max_tokens=max(N, max(lens)), max_pos=max(2 * N, 4096))
    if heads and world > 1:
        uid = D.broadcast_bytes(P.nccl_unique_id() if rank == 0 else b"", src=0)
        ctx.set_comm(uid, rank, world)
        if args.tp_comm == "p2p":  # NVLink peer-memory collectives instead of NCCL calls
            ctx.enable_tp_p2p()
            hs = [None] * world
            dist.all_gather_object(hs, ctx.tp_ipc_handle())
            ctx.tp_ipc_open(hs)
    if args.no_pdl:
        ctx.set_option("pdl", 0)
    for kv in filter(None, os.environ.get("CB_OPTS", "").split(",")):  # tuning: CB_OPTS=name=value,...
        k_, v_ = kv.split("=")
        ctx.set_option(k_, int(v_))
    mw = (P.ModelWeights.synth_shard(s, args.seed, "bf16", dev, rank, world) if heads and world > 1
          else P.ModelWeights.synth(s, args.seed, "bf16", dev))
    tok_h = req.tokens(s.vocab)
    tok = torch.from_numpy(tok_h).to(dev)
    pos = torch.from_numpy(req.global_positions()).to(dev)
    # chunk caches: standalone prefill of each chunk at local positions 0..L_c-1, produced by
    # this library (cb_blend_forward with the whole chunk as uncached suffix = full prefill)
    k_in = torch.empty(L, N, sh.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
    v_in = torch.empty_like(k_in)
    cs = req.chunk_starts()
    for c in range(len(lens)):
        a, b = int(cs[c]), int(cs[c + 1])
        n = b - a
        kc = torch.empty(L, n, sh.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
        vc = torch.empty_like(kc)
        P.blend_forward(ctx, mw, tok[a:b].contiguous(), torch.arange(n, dtype=torch.int32, device=dev), [0], n,
                        None, None, kc, vc, [0] * L)
        k_in[:, a:b] = kc
        v_in[:, a:b] = vc
    del kc, vc
    ks = P.schedule(ratio, N, L)
    k_out, v_out = torch.empty_like(k_in), torch.empty_like(v_in)
    h_out = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step_eager():
        P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, k_out, v_out, ks, h_out=h_out)

    l0 = ctx.launch_count()
    step_eager()  # also warms the tensor-map caches
    per_step_launches = ctx.launch_count() - l0
    torch.cuda.synchronize()
    step = step_eager
    if not args.no_graph:  # the whole blend as one CUDA graph (static shapes: every k_i is a host integer)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_eager()
        step = graph.replay
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof_range = os.environ.get("CB_PROFILE_RANGE") == "1"  # ncu --profile-from-start off: timed steps only
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if prof_range:
            torch.cuda.cudart().cudaProfilerStart()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if prof_range:
            torch.cuda.cudart().cudaProfilerStop()
    if world > 1:
        dist.barrier()
    launches = per_step_launches * args.steps
    ms = e0.elapsed_time(e1) / args.steps
    from paper_2405_16444_b200.dist import job_throughput, max_over_ranks
    if heads:  # one request over all ranks: its tokens / the slowest rank's time
        ms_max = max_over_ranks(ms, dev)
        value = N / (ms_max / 1e3)
    else:
        value, ms_max, _ = job_throughput(N, ms, dev)  # all ranks' tokens / slowest rank's time

    # end to end through the public API: chunk caches + tokens from pinned host memory, h_out back. Timed right
    # after the device-timed steps (before the profiling passes heat the GPU further), and the request path's
    # overhead over the device step is also measured paired (interleaved replays), free of that drift.
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(P, ctx, mw, req, s, ks, k_in, v_in, tok_h, dev, args, dev_step=step if world == 1 else None)
        if world > 1:
            e2e["value"] = (1 if heads else world) * N / (max_over_ranks(e2e["ms"], dev) / 1e3)

    if os.environ.get("CB_TRACE_SEL"):  # tuning: per-CTA event trace of the last matching launch of a step
        ctx.set_option("debug_trace", int(os.environ["CB_TRACE_SEL"]))
        step_eager()
        torch.cuda.synchronize()
        import ctypes
        raw = (ctypes.c_int64 * 2048)()
        P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 2048))
        np.save(os.environ.get("CB_TRACE_OUT", "gpurun_out/trace.npy"), np.array(raw[:], dtype=np.int64))
        ctx.set_option("debug_trace", 0)

    # per-kernel profile pass (same steps, per-launch CUDA events on the launching stream)
    prof = P.api.profile_steps(ctx, step_eager, max(3, min(args.steps, 10)))
    # the step's selections, for the exact attention FLOP count (one extra eager step, not timed)
    sel_t = torch.full((L, N), -1, dtype=torch.int32, device=dev)
    P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, k_out, v_out, ks, h_out=h_out, sel_out=sel_t)
    sel_np = sel_t.cpu().numpy()
    sel_sets = [row[row >= 0] for row in sel_np]
    work = algorithmic_work(sh, N, 0, ks, sel_sets)  # this rank's share (its heads / features) under heads
    hbm, tf_burst, tf_sus, peak_src = measured_peaks()
    gemm_ms = prof.get("gemm", 0.0)
    roof = None
    if gemm_ms > 0:
        achieved = work["gemm_flops"] / (gemm_ms / 1e3) / 1e12
        traffic, tnote = None, None
        for tname in ("r02g_traffic.json", "r02d_traffic.json", "r02_traffic.json", "r01c_traffic.json"):  # newest committed ncu capture first
            tpath = os.path.join(ROOT, "profiles", tname)
            if os.path.exists(tpath):  # committed ncu measurement of the largest GEMM launch (bytes per launch)
                tj = json.load(open(tpath))
                traffic = tj["dram_bytes"]
                tnote = (f"{tj['kernel']}: DRAM {tj['dram_bytes']} B vs algorithmic {tj['algorithmic_bytes']} B "
                         f"per launch ({tj['source']})")
                break
        attn_ms = prof.get("attention", 0.0)
        realign_ms = prof.get("realign", 0.0)
        roof = {"bound": "tensor", "kernel": "gemm (all projections)", "achieved": achieved, "peak": tf_burst,
                "unit": "TFLOP/s", "frac": achieved / tf_burst, "traffic": traffic, "traffic_note": tnote,
                "peak_source": f"{peak_src} bf16_tflops (burst; the step is ~10 ms of back-to-back kernels)",
                "frac_vs_sustained": achieved / tf_sus, "sustained_peak": tf_sus,
                "share_of_step": gemm_ms / ms,
                "attention": {"achieved": work["attn_flops"] / (attn_ms / 1e3) / 1e12 if attn_ms else None,
                              "frac": work["attn_flops"] / (attn_ms / 1e3) / 1e12 / tf_burst if attn_ms else None,
                              "flops": work["attn_flops"], "exact_spans": True},
                "realign": {"GBps_k_only": work["realign_k_bytes"] / (realign_ms / 1e3) / 1e9 if realign_ms else None,
                            "frac_k_only": work["realign_k_bytes"] / (realign_ms / 1e3) / 1e9 / hbm if realign_ms else None,
                            "frac_with_v_copy": work["realign_bytes"] / (realign_ms / 1e3) / 1e9 / hbm if realign_ms else None,
                            "hbm_peak": hbm},
                "path": path_roofline(work, prof, ms, hbm, tf_burst)}
    # the paper's comparison points on the same kernels and inputs -- full prefill (every
    # token recomputed: the whole request as uncached suffix) and full KV reuse (r = 0: realign + layer 0)
    baselines = None
    if not args.no_baselines:
        def timed(fn, n):
            g = torch.cuda.CUDAGraph()
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                fn()
            for _ in range(2):
                g.replay()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a_.record(stream)
            for _ in range(n):
                g.replay()
            b_.record(stream)
            torch.cuda.synchronize()
            return max_over_ranks(a_.elapsed_time(b_) / n, dev)
        h_full = torch.empty(N, s.d_model, dtype=torch.float32, device=dev)
        nb = max(3, min(args.steps, 10))
        ms_full = timed(lambda: P.blend_forward(ctx, mw, tok, pos, [0], N, None, None, k_out, v_out, [0] * L,
                                                h_out=h_full), nb)
        ks0 = [N] + [0] * (L - 1)
        ms_reuse = timed(lambda: P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, k_out, v_out, ks0,
                                                 h_out=h_full), nb)
        # prefix caching: only the first chunk's KV is reused (it IS a prefix, so exact); every
        # later token is prefilled -- the first chunk as cached context, the rest as the uncached suffix
        n0 = int(cs[1])
        k0, v0 = k_in[:, :n0].contiguous(), v_in[:, :n0].contiguous()  # the prefix chunk's cache, outside timing
        ms_prefix = timed(lambda: P.blend_forward(ctx, mw, tok, pos, [0, n0], N - n0, k0, v0, k_out, v_out,
                                                  [n0] + [0] * (L - 1), h_out=h_full), nb)
        del k0, v0
        del h_full
        baselines = {"full_prefill_ms": ms_full, "prefix_caching_ms": ms_prefix, "full_kv_reuse_ms": ms_reuse,
                     "blend_ms": ms_max, "blend_speedup_vs_full_prefill": ms_full / ms_max,
                     "blend_speedup_vs_prefix_caching": ms_prefix / ms_max,
                     "note": "same library kernels and inputs, one CUDA graph each; full prefill = every token "
                             "recomputed (no cache); prefix caching = the first chunk's KV reused, the other "
                             f"{len(lens) - 1} chunks prefilled (P:374-391); full KV reuse = r=0 (realign + full "
                             "layer 0 only). The paper quotes 2.2-3.3x TTFT vs full prefill on its GPUs (P:731), "
                             "context only"}
    # the loading controller for this request with the chunk KV in pinned
    # host memory: T_load from the measured host->HBM copy rate of one layer, Prefill from the full-prefill
    # baseline above (per layer), r = max(r_eq, 15 %)
    controller = None
    if baselines is not None:
        kv_tok = 2 * sh.n_kv_heads * s.head_dim * 2  # K and V of one token, one layer, bf16 (this rank's heads)
        host = torch.empty(N * kv_tok // 2, dtype=torch.bfloat16).pin_memory()
        devb = torch.empty_like(host, device=dev)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            devb.copy_(host, non_blocking=True)
        a_.record(stream)
        for _ in range(5):
            devb.copy_(host, non_blocking=True)
        b_.record(stream)
        torch.cuda.synchronize()
        bpm = 5 * host.numel() * 2 / a_.elapsed_time(b_)  # bytes per ms
        pre_layer = baselines["full_prefill_ms"] / L
        r_ctl, load_ms = P.api.controller_ratio(pre_layer, kv_tok, N, bpm, 0.15)
        controller = {"h2d_GBps": bpm / 1e6, "load_ms_per_layer": load_ms, "prefill_ms_per_layer": pre_layer,
                      "r": r_ctl, "r_eq": load_ms / pre_layer,
                      "note": "cb_controller_ratio: T_recompute(r) = r x Prefill per layer equals T_load per layer "
                              "(pinned host -> HBM), then max(r, 15%) (P:2693-2700)"}
        del host, devb
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = OracleSample(s, lens, ratio, args.seed)
        est, sample_s = smp.run()
        cpu = {"value": N / est, "unit": "ctx_tok/s", "cores": OracleSample.cores(), "kind": "oracle",
               "ms_per_blend": est * 1e3,
               "sample": f"realign all {L} layers + layers 0-2 in full (fp64 numpy, {sample_s:.1f} s); "
                         f"layers 3..{L - 1} extrapolated from layer 2 by row counts"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ctx_tok/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong" if heads else "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded counter RNG weights/tokens; "
                "chunk caches from standalone prefill of each chunk)",
                "config": {"workload": f"{shape_name} {len(lens)}x{lens[0]} tokens, r={ratio}, " +
                                       (f"1 request split by heads over {world} GPU(s)" if heads else "1 request per GPU"),
                           "recompute_ratio": ratio, "n_ctx": N, "k_sched_first_last": [ks[1], ks[-1]],
                           "parallelism": f"head-parallel tp{world} ({args.tp_comm} all-gather of Delta_kv partials, "
                                          "all-reduce after o_proj and down_proj)" if heads else
                                          f"request-parallel x{world}",
                           "l2": f"inputs larger than L2 ({work['weight_bytes'] / 1e9:.1f} GB of weights streamed "
                                 "per step per GPU)"},
                "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "baselines": baselines, "controller": controller,
                "kernel_ms": {k: round(v, 4) for k, v in prof.items()},
                "work": {k: float(v) for k, v in work.items()}}
    if heads and world > 1 and not args.no_request_sub:
        # the same job request-parallel (SURVEY §8(e) partitioning 2): every rank blends its own request on a
        # full replica, no collective -- measured after the head-parallel buffers are released
        step = step_eager = graph = None  # the closures hold the head-parallel buffers too
        del mw, k_in, v_in, k_out, v_out, ctx, step, step_eager, graph
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        sub = request_parallel_record(P, args, s, lens, ratio, world, rank, dev)
        if rank == 0:
            line["request_parallel"] = sub
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def request_parallel_record(P, args, s, lens, ratio, world, rank, dev):
    """Request-parallel measurement at N ranks (weak scaling): rank r blends request seed + r on its own full
    model replica; job value = all ranks' context tokens over the slowest rank's CUDA-event time."""
    import torch
    from paper_2405_16444_b200.dist import job_throughput
    req = W.Request(list(lens), 0, args.seed + rank, ratio)
    N, L = req.n_ctx, s.n_layers
    ctx = P.Context(s, "bf16", max_tokens=max(N, max(lens)), max_pos=max(2 * N, 4096))
    mw = P.ModelWeights.synth(s, args.seed, "bf16", dev)
    tok = torch.from_numpy(req.tokens(s.vocab)).to(dev)
    pos = torch.from_numpy(req.global_positions()).to(dev)
    cs = req.chunk_starts()
    k_in = torch.empty(L, N, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
    v_in = torch.empty_like(k_in)
    for c in range(len(lens)):
        a, b = int(cs[c]), int(cs[c + 1])
        kc = torch.empty(L, b - a, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
        vc = torch.empty_like(kc)
        P.blend_forward(ctx, mw, tok[a:b].contiguous(), torch.arange(b - a, dtype=torch.int32, device=dev), [0],
                        b - a, None, None, kc, vc, [0] * L)
        k_in[:, a:b] = kc
        v_in[:, a:b] = vc
    ks = P.schedule(ratio, N, L)
    k_out, v_out = torch.empty_like(k_in), torch.empty_like(v_in)
    h_out = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=dev)
    fn = lambda: P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, k_out, v_out, ks, h_out=h_out)
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    import torch.distributed as dist
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    value, ms_max, tok_all = job_throughput(N, e0.elapsed_time(e1) / args.steps, dev)
    return {"value": value, "unit": "ctx_tok/s", "ms_per_step": ms_max, "scaling": "weak", "ctx_tokens": tok_all,
            "parallelism": f"request-parallel x{world} (one request per GPU, full replica, no collective)"}


def run_e2e(P, ctx, mw, req, s, ks, k_in, v_in, tok_h, dev, args, dev_step=None):
    import torch
    N, L = req.n_ctx, s.n_layers
    kh = k_in.cpu().pin_memory()
    vh = v_in.cpu().pin_memory()
    toks = torch.from_numpy(tok_h).pin_memory()
    poss = torch.from_numpy(req.global_positions()).pin_memory()
    hh = torch.empty(ks[-1], s.d_model, dtype=torch.float32).pin_memory()
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    cs = list(req.chunk_starts())
    stream = torch.cuda.current_stream()

    def step_eager():
        P.api.blend_request(ctx, mw, toks, poss, cs, 0, kh, vh, kb, vb, ks, hh)

    step_eager()
    torch.cuda.synchronize()
    step, graphed = step_eager, False
    if not args.no_graph:  # copy stream forks/joins inside the capture through the library's events
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step_eager()
            step, graphed = graph.replay, True
        except Exception:
            torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    paired = None
    if dev_step is not None and graphed:  # interleaved single replays: request path minus device step
        diffs = []
        for r in range(2 * max(5, args.steps)):
            t = {}
            for name, fn in ((("req", step), ("dev", dev_step)) if r % 2 == 0 else (("dev", dev_step), ("req", step))):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                t[name] = a.elapsed_time(b)
            diffs.append(t["req"] - t["dev"])
        paired = float(np.median(diffs))
    h2d = kh.numel() * 2 + vh.numel() * 2 + toks.numel() * 4 + poss.numel() * 4
    d2h = hh.numel() * 4
    return {"value": N / (ms / 1e3), "unit": "ctx_tok/s", "ms": ms, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "paired_overhead_ms": paired,
            "path": "cb_blend_request: pinned host chunk KV + tokens, layer-pipelined H2D on a copy stream, "
                    "h_out D2H; KV^new stays on the GPU" + (" (CUDA graph)" if graphed else "")}


def run_attn_deviation(args):
    """SURVEY §8(f) N2 on the GPU path: attention deviation Delta_attn(A_i, A_i^full) (reading R16) of
    a request with a 32-token query suffix, per recompute ratio, for the HKVD selection (the blend's own top-k)
    and for a random nested selection of the same sizes (Fig. ca_reduction). Every layer runs through
    cb_blend_layer (library kernels); the suffix rows' queries and the attention matrices of this analysis are
    formed from the layer outputs with torch (fp32) -- measurement code, not the blend path."""
    import torch
    import paper_2405_16444_b200 as P
    from paper_2405_16444_b200.build import build
    build()
    shape_name, lens, _ = CONFIGS[args.config if args.config in CONFIGS else "mistral"]
    s = W.MODELS[shape_name]
    n_suf = 32
    req = W.Request(list(lens), n_suf, args.seed, 0.15)
    N, T, L = req.n_ctx, req.n_total, s.n_layers
    qd, hd = s.qd, s.head_dim
    dev = torch.device("cuda", 0)
    ctx = P.Context(s, "bf16", max_tokens=T, max_pos=max(2 * T, 4096))
    mw = P.ModelWeights.synth(s, args.seed, "bf16", dev)
    tok = torch.from_numpy(req.tokens(s.vocab)).to(dev)
    pos = torch.from_numpy(req.global_positions()).to(dev)
    cs = req.chunk_starts()
    k_in = torch.empty(L, N, s.n_kv_heads, hd, dtype=torch.bfloat16, device=dev)
    v_in = torch.empty_like(k_in)
    for c in range(len(lens)):  # chunk caches: standalone prefill of each chunk at local positions
        a, b = int(cs[c]), int(cs[c + 1])
        kc = torch.empty(L, b - a, s.n_kv_heads, hd, dtype=torch.bfloat16, device=dev)
        vc = torch.empty_like(kc)
        P.blend_forward(ctx, mw, tok[a:b].contiguous(), torch.arange(b - a, dtype=torch.int32, device=dev), [0],
                        b - a, None, None, kc, vc, [0] * L)
        k_in[:, a:b] = kc
        v_in[:, a:b] = vc
    inv = 1.0 / (s.rope_theta ** (torch.arange(0, hd, 2, device=dev, dtype=torch.float64) / hd))
    qpos = pos[N:].double()
    ang = qpos[:, None] * inv[None, :]
    cos, sin = torch.cos(ang).float(), torch.sin(ang).float()
    G = s.n_q_heads // s.n_kv_heads

    def attn_matrix(i, h_suf, kb):
        """A_i of the suffix rows: softmax(q K^T / sqrt(hd)) over all T keys, masked by position, [n_q][32][T]."""
        w = mw.layers[i]
        x = h_suf * torch.rsqrt(h_suf.pow(2).mean(-1, keepdim=True) + s.rms_eps) * w["attn_norm"]
        q = (x @ w["w_qkv"][:qd].float().T).view(n_suf, s.n_q_heads, hd)
        q0, q1 = q[..., 0::2], q[..., 1::2]  # interleaved pairs (2i, 2i+1), R9
        qr = torch.empty_like(q)
        qr[..., 0::2] = q0 * cos[:, None] - q1 * sin[:, None]
        qr[..., 1::2] = q0 * sin[:, None] + q1 * cos[:, None]
        k = kb.float().repeat_interleave(G, dim=1)  # [T][n_q][hd]
        sc = torch.einsum("rhd,thd->hrt", qr, k) / math.sqrt(hd)
        mask = pos[None, :] > pos[N:][:, None]  # key after the query: hidden
        sc = sc.masked_fill(mask[None], float("-inf"))
        return torch.softmax(sc, dim=-1)

    def stepped(ks, force=None, full=False):
        """Per layer: the suffix rows' input h and this layer's blended K after the layer ran."""
        kb = torch.empty(L, T, s.n_kv_heads, hd, dtype=torch.bfloat16, device=dev)
        vb = torch.empty_like(kb)
        if not full:
            kb[:, :N] = k_in
            vb[:, :N] = v_in
            loc = torch.from_numpy(np.concatenate([req.local_positions(), np.zeros(n_suf)]).astype(np.int32)).to(dev)
            P.rope_realign(ctx, kb, kb, loc, pos, L, T, T * s.kvd)
        h = P.api.op_embed(ctx, mw.embed, tok)
        Nn = 0 if full else N
        cand = torch.arange(Nn, dtype=torch.int32, device=dev)
        outs = []
        for i in range(L):
            nc = cand.numel()
            h_suf = h[nc:nc + (T - Nn if full else n_suf)][-n_suf:].clone()
            if i == 0:
                P.blend_layer(ctx, 0, mw, h, cand, Nn, T - Nn if full else n_suf, kb[0], vb[0], pos, Nn)
            else:
                fs = None if force is None else torch.from_numpy(force[i].astype(np.int32)).to(dev)
                sel, _ = P.blend_layer(ctx, i, mw, h, cand, 0 if full else ks[i], T - Nn if full else n_suf, kb[i],
                                       vb[i], pos, Nn, force_sel=fs)
                cand = sel.clone()
            outs.append((h_suf, kb[i]))
        return outs

    full = stepped(None, full=True)
    a_full = [attn_matrix(i, hs, kb) for i, (hs, kb) in enumerate(full)]
    ratios = [0.0, 0.05, 0.1, 0.15, 0.2, 0.3, 0.5, 1.0]
    curve = {"hkvd": [], "random": []}
    for r in ratios:
        ks = P.schedule(r, N, L)
        for mode in ("hkvd", "random"):
            force = W.nested_selection(args.seed + 100, N, ks) if mode == "random" else None
            out = stepped(ks, force=force)
            d = [float(torch.linalg.vector_norm(attn_matrix(i, hs, kb) - a_full[i])) for i, (hs, kb) in enumerate(out)]
            curve[mode].append(float(np.mean(d[1:])))
    torch.cuda.synchronize()
    print(json.dumps({"kind": "attention deviation (P:119-121, R16), mean over layers 1..L-1",
                      "workload": f"{shape_name} {len(lens)}x{lens[0]} + {n_suf}-token query suffix, random-init weights",
                      "ratios": ratios, "hkvd": curve["hkvd"], "random": curve["random"],
                      "note": "blend layers through cb_blend_layer (HKVD = the library's own top-k; random = a seeded "
                              "nested selection of the same k_i as force_sel); full prefill = the same request as "
                              "an uncached all-suffix blend; A_i of the suffix rows formed with torch fp32"}), flush=True)


def run_batched(args):
    """independent Mistral-shape requests, longest-first over the ranks, each rank
    blending its own requests back to back (one CUDA graph per request). Weak scaling, no collective on
    the data path; the job throughput is all ranks' context tokens over the slowest rank's time."""
    import torch
    import torch.distributed as dist

    from paper_2405_16444_b200.dist import assign_requests, job_throughput, world_info
    rank, world, local = world_info()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2405_16444_b200.build import build
    if rank == 0 or world == 1:
        build()
    if world > 1:
        dist.barrier()
    import paper_2405_16444_b200 as P
    reqs = W.config_requests("batched", args.seed)[:args.batched_requests]
    parts = assign_requests([r.n_ctx for r in reqs], world)
    mine = [reqs[i] for i in parts[rank]]
    s = W.MODELS["mistral-7b"]
    dev = torch.device("cuda", local)
    L = s.n_layers
    Nmax = max(r.n_ctx for r in mine) if mine else 1
    ctx = P.Context(s, "bf16", max_tokens=Nmax, max_pos=max(2 * Nmax, 4096))
    mw = P.ModelWeights.synth(s, args.seed, "bf16", dev)
    graphs, tokens = [], 0
    for req in mine:
        N = req.n_ctx
        tok = torch.from_numpy(req.tokens(s.vocab)).to(dev)
        pos = torch.from_numpy(req.global_positions()).to(dev)
        cs = req.chunk_starts()
        k_in = torch.empty(L, N, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
        v_in = torch.empty_like(k_in)
        for c in range(len(cs) - 1):  # the request's chunk caches (standalone prefill)
            a, b = int(cs[c]), int(cs[c + 1])
            kc = torch.empty(L, b - a, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=dev)
            vc = torch.empty_like(kc)
            P.blend_forward(ctx, mw, tok[a:b].contiguous(), torch.arange(b - a, dtype=torch.int32, device=dev), [0],
                            b - a, None, None, kc, vc, [0] * L)
            k_in[:, a:b] = kc
            v_in[:, a:b] = vc
        ks = P.schedule(req.ratio, N, L)
        kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
        h_out = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=dev)

        def step(tok=tok, pos=pos, cs=cs, k_in=k_in, v_in=v_in, kb=kb, vb=vb, ks=ks, h_out=h_out):
            P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, kb, vb, ks, h_out=h_out)
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        graphs.append((g, step))  # the closure keeps the request's buffers alive for the replays
        tokens += N
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for g, _ in graphs:
            g.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            for g, _ in graphs:
                g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    value, ms_max, tok_all = job_throughput(tokens, ms, dev)
    if rank == 0:
        loads = [sum(reqs[i].n_ctx for i in p) for p in parts]
        print(json.dumps({
            "metric": "context tok/s of independent blend requests (SURVEY config 5)", "value": value,
            "unit": "ctx_tok/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter RNG weights/tokens; chunk caches from standalone prefill)",
            "config": {"workload": f"batched: {len(reqs)} mistral-7b requests, 4-8 chunks x 256-1024 tokens, r=0.15",
                       "parallelism": f"request-parallel x{world} (longest-first)", "ctx_tokens": int(tok_all),
                       "rank_tokens": loads, "balance": max(loads) / (sum(loads) / len(loads))},
            "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.cpu_full:
        run_cpu_full(a)
    elif a.attn_deviation:
        run_attn_deviation(a)
    elif a.impl == "reference":
        run_reference(a)
    elif a.config == "batched":
        run_batched(a)
    else:
        run_ours(a)
