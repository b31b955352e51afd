"""Thin Python binding of libcacheblend (same names as the C-ABI; argument marshalling only).

PyTorch provides device memory, streams and process groups; every step of the blend runs in the
library's sm_100a kernels. Nothing here computes any part of the method."""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from ._lib import CbLayerW, CbModel, CacheBlendError, check, lib

DTYPES = {"bf16": 0, "f32": 1}
TORCH_DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _i32(seq: Sequence[int]):
    arr = (ctypes.c_int32 * len(seq))(*[int(x) for x in seq])
    return arr


class Context:
    """cb_ctx owner. `shape` is any object with the synth.workload.ModelShape fields."""

    def __init__(self, shape, dtype: str, max_tokens: int, max_pos: Optional[int] = None,
                 device: Optional[torch.device] = None):
        self.shape, self.dtype, self.max_tokens = shape, dtype, int(max_tokens)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.m = CbModel(shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                         shape.d_ff, shape.vocab, float(shape.rope_theta), float(shape.rms_eps), DTYPES[dtype],
                         int(max_pos if max_pos is not None else max(2 * max_tokens, 16)))
        nbytes = ctypes.c_size_t(0)
        check(lib().cb_workspace_size(ctypes.byref(self.m), self.max_tokens, ctypes.byref(nbytes)))
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
            h = ctypes.c_void_p()
            check(lib().cb_create(ctypes.byref(self.m), self.max_tokens, self.workspace.data_ptr(), nbytes.value,
                                  ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().cb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check_device_errors(self):
        check(lib().cb_check_device_errors(self.handle))

    def launch_count(self) -> int:
        return int(lib().cb_launch_count(self.handle))

    def set_option(self, name: str, value: int):
        check(lib().cb_set_option(self.handle, name.encode(), int(value)))

    def set_comm(self, uid: bytes, rank: int, world: int):
        """Join an NCCL communicator for the head-parallel blend (cb_set_comm). The context must have been
        created with dist.head_shard_shape(shape, world)."""
        assert len(uid) == 128
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        with torch.cuda.device(self.device):
            check(lib().cb_set_comm(self.handle, buf, int(rank), int(world)))
        self.tp = (int(rank), int(world))

    def set_comm_local(self, group: "Group", rank: int):
        """Join a one-process loopback group (cb_set_comm_local; tests of the head-parallel path on one GPU)."""
        with torch.cuda.device(self.device):
            check(lib().cb_set_comm_local(self.handle, group.handle, int(rank)))
        self.tp = (int(rank), group.world)
        self._group = group  # the group must outlive the context

    def enable_tp_p2p(self):
        """NVLink peer-memory collectives (cb_tp_p2p_enable) after set_comm / set_comm_local."""
        with torch.cuda.device(self.device):
            check(lib().cb_tp_p2p_enable(self.handle))

    def tp_ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib().cb_tp_ipc_handle(self.handle, buf))
        return buf.raw

    def tp_ipc_open(self, handles: Sequence[bytes]):
        """handles: every rank's tp_ipc_handle() in rank order."""
        blob = b"".join(bytes(h) for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        with torch.cuda.device(self.device):
            check(lib().cb_tp_ipc_open(self.handle, buf))

    def info(self, name: str) -> int:
        v = ctypes.c_int64(0)
        check(lib().cb_get_info(self.handle, name.encode(), ctypes.byref(v)))
        return v.value


class Group:
    """cb_group: loopback head-parallel group of `world` contexts in this process (cb_group_create)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        check(lib().cb_group_create(int(world), ctypes.byref(h)))
        self.handle, self.world = h, int(world)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().cb_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().cb_nccl_unique_id(buf))
    return buf.raw


class ModelWeights:
    """Device weights in the C-ABI layouts (cacheblend.h cb_layer_w)."""

    def __init__(self, shape, dtype: str, embed: torch.Tensor, layers: List[Dict[str, torch.Tensor]]):
        self.shape, self.dtype, self.embed, self.layers = shape, dtype, embed, layers
        self.cw = (CbLayerW * shape.n_layers)()
        for i, w in enumerate(layers):
            self.cw[i] = CbLayerW(_p(w["attn_norm"]), _p(w["w_qkv"]), _p(w["w_o"]), _p(w["mlp_norm"]),
                                  _p(w["w_gate_up"]), _p(w["w_down"]))

    @staticmethod
    def empty(shape, dtype: str, device) -> "ModelWeights":
        td = TORCH_DTYPES[dtype]
        d, qd, kvd, ff = shape.d_model, shape.n_q_heads * shape.head_dim, shape.n_kv_heads * shape.head_dim, shape.d_ff
        layers = []
        for _ in range(shape.n_layers):
            layers.append({
                "attn_norm": torch.empty(d, dtype=torch.float32, device=device),
                "w_qkv": torch.empty(qd + 2 * kvd, d, dtype=td, device=device),
                "w_o": torch.empty(d, qd, dtype=td, device=device),
                "mlp_norm": torch.empty(d, dtype=torch.float32, device=device),
                "w_gate_up": torch.empty(2 * ff, d, dtype=td, device=device),
                "w_down": torch.empty(d, ff, dtype=td, device=device),
            })
        return ModelWeights(shape, dtype, torch.empty(shape.vocab, d, dtype=td, device=device), layers)

    @staticmethod
    def synth(shape, seed: int, dtype: str, device, layer_ids: Optional[Sequence[int]] = None) -> "ModelWeights":
        """Fill with the synth.workload recipe through the library's counter RNG (cb_gen_fill). layer_ids:
        which model layers the shape's layers hold (default 0..n_layers-1)."""
        from synth import workload as W
        mw = ModelWeights.empty(shape, dtype, device)
        ids = list(range(shape.n_layers)) if layer_ids is None else list(layer_ids)
        s = _stream(None)

        def fill(t: torch.Tensor, rec, row0: int = 0, is_f32: bool = False):
            dst = t.data_ptr() + row0 * t.shape[-1] * t.element_size() if t.dim() > 1 else t.data_ptr()
            check(lib().cb_gen_fill(dst, 1 if is_f32 else DTYPES[dtype], rec.count, seed, rec.stream, 0,
                                    rec.scale, rec.offset, s))

        fill(mw.embed, W.embed_recipe(shape))
        qd, kvd, ff = shape.n_q_heads * shape.head_dim, shape.n_kv_heads * shape.head_dim, shape.d_ff
        for i, w in zip(ids, mw.layers):
            r = W.layer_recipes(shape, i)
            fill(w["attn_norm"], r["attn_norm"], is_f32=True)
            fill(w["mlp_norm"], r["mlp_norm"], is_f32=True)
            fill(w["w_qkv"], r["wq"], 0)
            fill(w["w_qkv"], r["wk"], qd)
            fill(w["w_qkv"], r["wv"], qd + kvd)
            fill(w["w_o"], r["wo"])
            fill(w["w_gate_up"], r["wg"], 0)
            fill(w["w_gate_up"], r["wu"], ff)
            fill(w["w_down"], r["wd"])
        return mw

    @staticmethod
    def synth_shard(shape, seed: int, dtype: str, device, rank: int, world: int) -> "ModelWeights":
        """Rank's head-parallel shard of the synth recipe: each layer is generated in full (cb_gen_fill, one
        layer at a time) and sliced with dist.shard_layer. Returns weights of dist.head_shard_shape."""
        from . import dist as D
        one = dataclasses.replace(shape, n_layers=1)
        layers, embed = [], None
        for i in range(shape.n_layers):
            full = ModelWeights.synth(one, seed, dtype, device, layer_ids=[i])
            if embed is None:
                embed = full.embed
            layers.append(D.shard_layer(full.layers[0], shape, rank, world))
            del full
        return ModelWeights(D.head_shard_shape(shape, world), dtype, embed, layers)

    @staticmethod
    def from_host(shape, dtype: str, embed: np.ndarray, layers: List[Dict[str, np.ndarray]], device) -> "ModelWeights":
        """Upload oracle-side weight dicts (wq/wk/wv/wo/wg/wu/wd/attn_norm/mlp_norm) into the ABI layout."""
        td = TORCH_DTYPES[dtype]
        up = lambda a, dt=td: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device=device, dtype=dt)
        L = []
        for w in layers:
            L.append({"attn_norm": up(w["attn_norm"], torch.float32), "mlp_norm": up(w["mlp_norm"], torch.float32),
                      "w_qkv": up(np.concatenate([w["wq"], w["wk"], w["wv"]], 0)), "w_o": up(w["wo"]),
                      "w_gate_up": up(np.concatenate([w["wg"], w["wu"]], 0)), "w_down": up(w["wd"])})
        return ModelWeights(shape, dtype, up(embed), L)


def gen_fill(out: torch.Tensor, seed: int, stream_id: int, scale: float, offset: float = 0.0, start: int = 0):
    dt = 0 if out.dtype == torch.bfloat16 else 1
    check(lib().cb_gen_fill(out.data_ptr(), dt, out.numel(), seed, stream_id, start, scale, offset, _stream(None)))


def gen_ints(out: torch.Tensor, seed: int, stream_id: int, modulus: int, start: int = 0):
    assert out.dtype == torch.int32
    check(lib().cb_gen_ints(out.data_ptr(), out.numel(), seed, stream_id, start, modulus, _stream(None)))


# ---- the boundary calls -------------------------------------------------------------------------------
def schedule(ratio: float, n_ctx: int, n_layers: int) -> List[int]:
    out = (ctypes.c_int32 * n_layers)()
    check(lib().cb_schedule(float(ratio), int(n_ctx), int(n_layers), out))
    return list(out)


def kv_to_paged(ctx: Context, k_blend: torch.Tensor, v_blend: torch.Tensor, block_table: torch.Tensor,
                block_size: int, k_pages: torch.Tensor, v_pages: torch.Tensor, n_tok: Optional[int] = None,
                stream=None):
    """cb_kv_to_paged: k_blend/v_blend [L][T][n_kv][hd] -> k_pages/v_pages [L][n_pages][block_size][n_kv][hd]."""
    L, T = k_blend.shape[0], k_blend.shape[1]
    n = T if n_tok is None else int(n_tok)
    check(lib().cb_kv_to_paged(ctx.handle, _p(k_blend), _p(v_blend), L, n, k_blend[0].numel(), _p(block_table),
                               int(block_size), _p(k_pages), _p(v_pages), int(k_pages.shape[1]), k_pages[0].numel(),
                               _stream(stream)))


def chunk_digest(model_id: bytes, tokens) -> bytes:
    """cb_chunk_digest: the chunk's 32-byte store key, SHA-256 of (len(model_id) as u32 LE || model_id ||
    token ids as LE int32) (host)."""
    a = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
    mid = bytes(model_id)
    out = ctypes.create_string_buffer(32)
    check(lib().cb_chunk_digest(mid, len(mid), a.ctypes.data if a.size else None, a.size, out))
    return out.raw


def model_identity(shape, dtype: str, weights_id: str) -> bytes:
    """A model id for chunk_digest: the model configuration plus the caller's weights identifier (e.g. the
    checkpoint's hash, or the synthetic recipe and seed)."""
    f = (shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, shape.d_ff, shape.vocab,
         float(shape.rope_theta), float(shape.rms_eps), dtype, weights_id)
    return repr(f).encode()


def _key(key: bytes):
    b = bytes(key)
    if len(b) != 32:
        raise ValueError("a store key is a 32-byte chunk_digest")
    return ctypes.create_string_buffer(b, 32)


class Store:
    """cb_store: chunk hash -> chunk KV (host RAM, LRU eviction)."""

    def __init__(self, capacity_bytes: int, pinned: bool = True):
        h = ctypes.c_void_p()
        check(lib().cb_store_create(int(capacity_bytes), int(pinned), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().cb_store_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def put(self, key: bytes, k: torch.Tensor, v: torch.Tensor):
        """key: chunk_digest(...) (32 bytes); k, v: [L][n_tok][n_kv][hd] (host or device, contiguous)."""
        assert k.is_contiguous() and v.is_contiguous() and k.shape == v.shape
        check(lib().cb_store_put(self.handle, _key(key), k.data_ptr(), v.data_ptr(), k.numel() * k.element_size(),
                                 int(k.shape[1])))

    def lookup(self, key: bytes, touch: bool = True) -> int:
        n = ctypes.c_int32(0)
        check(lib().cb_store_lookup(self.handle, _key(key), int(touch), ctypes.byref(n), None, None))
        return n.value

    def stats(self) -> Dict[str, int]:
        o = (ctypes.c_int64 * 6)()
        check(lib().cb_store_stats(self.handle, o))
        return dict(zip(("used", "capacity", "entries", "hits", "misses", "evictions"), list(o)))

    def set_disk(self, directory: str, capacity_bytes: int):
        """A disk level under `directory` (cb_store_set_disk): RAM evictions spill there; lookups read back."""
        check(lib().cb_store_set_disk(self.handle, str(directory).encode(), int(capacity_bytes)))

    def disk_stats(self) -> Dict[str, int]:
        o = (ctypes.c_int64 * 6)()
        check(lib().cb_store_disk_stats(self.handle, o))
        return dict(zip(("used", "capacity", "entries", "hits", "spills", "evictions"), list(o)))

    def get(self, key: bytes, shape, dtype) -> Optional[tuple]:
        """(k, v) host copies of the entry (promoted from disk if there), or None on a miss. shape: [L][n_tok][n_kv][hd]
        with n_tok (or any dimension) given as -1 = the entry's token count."""
        n = ctypes.c_int32(0)
        kp, vp = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib().cb_store_lookup(self.handle, _key(key), 1, ctypes.byref(n), ctypes.byref(kp), ctypes.byref(vp)))
        if n.value < 0:
            return None
        shape = tuple(n.value if d == -1 else d for d in shape)  # -1: the entry's token count
        count = int(np.prod(shape))
        nbytes = count * torch.empty(0, dtype=dtype).element_size()
        out = []
        for ptr in (kp.value, vp.value):
            buf = (ctypes.c_char * nbytes).from_address(ptr)
            out.append(torch.frombuffer(bytearray(buf), dtype=dtype).reshape(shape))
        return tuple(out)

    def keys(self) -> List[bytes]:
        n = ctypes.c_int32(0)
        check(lib().cb_store_keys(self.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(32 * max(n.value, 1))
        check(lib().cb_store_keys(self.handle, buf, n.value, ctypes.byref(n)))
        return [buf.raw[32 * i:32 * (i + 1)] for i in range(n.value)]


def blend_request_store(ctx: Context, store: Store, chunk_keys: Sequence[bytes], weights: ModelWeights,
                        tok_host: torch.Tensor, pos_host: torch.Tensor, chunk_start: Sequence[int], n_suffix: int,
                        k_blend: torch.Tensor, v_blend: torch.Tensor, k_sched: Sequence[int],
                        h_out_host: torch.Tensor, sel_out_host: Optional[torch.Tensor] = None, stream=None):
    """cb_blend_request_store: chunk KV fetched from the store layer by layer."""
    N = int(chunk_start[-1])
    blob = b"".join(_key(k).raw for k in chunk_keys)
    keys = ctypes.create_string_buffer(blob, max(len(blob), 32))
    check(lib().cb_blend_request_store(ctx.handle, store.handle, keys, weights.cw, _p(weights.embed), _p(tok_host),
                                       _p(pos_host), N, n_suffix, _i32(chunk_start), len(chunk_start) - 1,
                                       _p(k_blend), _p(v_blend), _i32(k_sched), _p(sel_out_host), _p(h_out_host),
                                       _stream(stream)))


def controller_ratio(prefill_ms: float, kv_bytes_per_token: float, n_tokens: int, bytes_per_ms: float,
                     r_min: float = 0.15):
    """Loading controller (cb_controller_ratio): (recompute ratio, T_load in ms) for one layer."""
    r, ld = ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(lib().cb_controller_ratio(float(prefill_ms), float(kv_bytes_per_token), int(n_tokens), float(bytes_per_ms),
                                    float(r_min), ctypes.byref(r), ctypes.byref(ld)))
    return r.value, ld.value


def controller_schedule(prefill_ms: float, kv_bytes_per_token: float, bytes_per_ms: float, n_ctx: int,
                        n_layers: int, r_min: float = 0.15):
    """cb_controller_schedule: (k_sched, r, T_load ms) -- the controller's ratio turned into per-layer counts."""
    k = (ctypes.c_int32 * n_layers)()
    r, ld = ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(lib().cb_controller_schedule(float(prefill_ms), float(kv_bytes_per_token), float(bytes_per_ms),
                                       float(r_min), int(n_ctx), int(n_layers), k, ctypes.byref(r), ctypes.byref(ld)))
    return list(k), r.value, ld.value


def controller_pick_device(prefill_ms: float, load_ms: Sequence[float], cost: Sequence[float],
                           r_fixed: float = 0.15) -> int:
    """cb_controller_pick_device: index of the cheapest storage device whose load is hidden, or -1."""
    n = len(load_ms)
    lm, co = (ctypes.c_double * max(n, 1))(*load_ms), (ctypes.c_double * max(n, 1))(*cost)
    out = ctypes.c_int32(0)
    check(lib().cb_controller_pick_device(float(prefill_ms), lm, co, n, float(r_fixed), ctypes.byref(out)))
    return out.value


def rope_realign(ctx: Context, k_out: torch.Tensor, k_src: torch.Tensor, src_pos: torch.Tensor,
                 dst_pos: torch.Tensor, n_slices: int, n_tok: int, slice_stride: int, stream=None):
    check(lib().cb_rope_realign(ctx.handle, _p(k_out), _p(k_src), _p(src_pos), _p(dst_pos), n_slices, n_tok,
                                slice_stride, _stream(stream)))


def kv_deviation_topk(ctx: Context, k_new, v_new, k_ref, v_ref, cand_tok: torch.Tensor, k_keep: int,
                      dev_mode: int = 0, want_dev: bool = True, stream=None):
    n = cand_tok.numel()
    dev = cand_tok.new_empty(n, dtype=torch.float32) if want_dev else None
    sel_tok = cand_tok.new_empty(max(k_keep, 1), dtype=torch.int32)
    sel_slot = cand_tok.new_empty(max(k_keep, 1), dtype=torch.int32)
    check(lib().cb_kv_deviation_topk(ctx.handle, _p(k_new), _p(v_new), _p(k_ref), _p(v_ref), _p(cand_tok), n,
                                     k_keep, dev_mode, _p(sel_tok), _p(sel_slot), _p(dev), _stream(stream)))
    return sel_tok[:k_keep], sel_slot[:k_keep], dev


def blend_layer(ctx: Context, layer: int, weights: ModelWeights, h: torch.Tensor, cand_tok: torch.Tensor,
                k_keep: int, n_suffix: int, k_blend: torch.Tensor, v_blend: torch.Tensor, pos: torch.Tensor, N: int,
                force_sel: Optional[torch.Tensor] = None, want_dev: bool = False, stream=None):
    n_cand = cand_tok.numel()
    sel = pos.new_empty(max(k_keep, 1), dtype=torch.int32)
    dev = pos.new_empty(max(n_cand, 1), dtype=torch.float32) if want_dev else None
    check(lib().cb_blend_layer(ctx.handle, layer, ctypes.byref(weights.cw[layer]), _p(h), _p(cand_tok), n_cand,
                               k_keep, n_suffix, _p(k_blend), _p(v_blend), _p(pos), N, _p(force_sel), _p(sel),
                               _p(dev), _stream(stream)))
    return sel[:k_keep], (dev[:n_cand] if dev is not None else None)


def blend_forward(ctx: Context, weights: ModelWeights, tok: torch.Tensor, pos: torch.Tensor,
                  chunk_start: Sequence[int], n_suffix: int, k_in: torch.Tensor, v_in: torch.Tensor,
                  k_blend: torch.Tensor, v_blend: torch.Tensor, k_sched: Sequence[int],
                  force_sel: Optional[torch.Tensor] = None, sel_out: Optional[torch.Tensor] = None,
                  dev_out: Optional[torch.Tensor] = None, h_out: Optional[torch.Tensor] = None, stream=None):
    """Runs cb_blend_forward; returns h_out (fp32 [k_{L-1} + n_suffix][d])."""
    N = int(chunk_start[-1])
    L = weights.shape.n_layers
    rows = (N if L == 1 else int(k_sched[-1])) + n_suffix
    if h_out is None:
        h_out = torch.empty(max(rows, 1), weights.shape.d_model, dtype=torch.float32, device=pos.device)
    cs = _i32(chunk_start)
    ks = _i32(k_sched)
    check(lib().cb_blend_forward(ctx.handle, weights.cw, _p(weights.embed), _p(tok), _p(pos), N, n_suffix, cs,
                                 len(chunk_start) - 1, _p(k_in), _p(v_in), _p(k_blend), _p(v_blend), ks,
                                 _p(force_sel), _p(sel_out), _p(dev_out), _p(h_out), _stream(stream)))
    return h_out[:rows]


def blend_request(ctx: Context, weights: ModelWeights, tok_host: torch.Tensor, pos_host: torch.Tensor,
                  chunk_start: Sequence[int], n_suffix: int, k_in_host: torch.Tensor, v_in_host: torch.Tensor,
                  k_blend: torch.Tensor, v_blend: torch.Tensor, k_sched: Sequence[int], h_out_host: torch.Tensor,
                  sel_out_host: Optional[torch.Tensor] = None, stream=None):
    """cb_blend_request: inputs in (pinned) host memory, KV^new on the device, h_out back in host memory."""
    N = int(chunk_start[-1])
    check(lib().cb_blend_request(ctx.handle, weights.cw, _p(weights.embed), _p(tok_host), _p(pos_host), N, n_suffix,
                                 _i32(chunk_start), len(chunk_start) - 1, _p(k_in_host), _p(v_in_host), _p(k_blend),
                                 _p(v_blend), _i32(k_sched), _p(sel_out_host), _p(h_out_host), _stream(stream)))


def profile_steps(ctx: Context, step, n: int) -> Dict[str, float]:
    """Runs `step` n times with per-launch CUDA events; returns device ms per step for each kernel class."""
    N_CLS = 10
    check(lib().cb_profile_begin(ctx.handle))
    for _ in range(n):
        step()
    ms = (ctypes.c_double * N_CLS)()
    cnt = (ctypes.c_int64 * N_CLS)()
    check(lib().cb_profile_end(ctx.handle, ms, cnt, N_CLS))
    return {lib().cb_profile_class_name(i).decode(): ms[i] / n for i in range(N_CLS) if cnt[i]}


def op_gemm(ctx: Context, A: torch.Tensor, B: torch.Tensor, out_f32: bool = False, impl: int = 0, stream=None):
    M, K = A.shape
    N = B.shape[0]
    C = A.new_empty(M, N, dtype=torch.float32 if out_f32 else A.dtype)
    check(lib().cb_op_gemm(ctx.handle, _p(A), _p(B), _p(C), M, N, K, int(out_f32), impl, _stream(stream)))
    return C


def op_gemm_resid(ctx: Context, A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, impl: int = 0, stream=None):
    """In place C += A . B^T on an fp32 C (the residual epilogue of the o-/down-projections)."""
    M, K = A.shape
    N = B.shape[0]
    assert C.dtype == torch.float32 and C.shape == (M, N) and C.is_contiguous()
    check(lib().cb_op_gemm(ctx.handle, _p(A), _p(B), _p(C), M, N, K, 2, impl, _stream(stream)))
    return C


def op_attention(ctx: Context, q, q_row, q_tok, k, v, n_keys: int, impl: int = 0, stream=None):
    n = q_row.numel()
    out = q.new_empty(n, ctx.shape.n_q_heads * ctx.shape.head_dim)
    check(lib().cb_op_attention(ctx.handle, _p(q), _p(q_row), _p(q_tok), n, _p(k), _p(v), n_keys, _p(out), impl,
                                _stream(stream)))
    return out


def op_rmsnorm(ctx: Context, h: torch.Tensor, gain: torch.Tensor, stream=None):
    x = h.new_empty(h.shape, dtype=TORCH_DTYPES[ctx.dtype])
    check(lib().cb_op_rmsnorm(ctx.handle, _p(h), _p(gain), h.shape[0], _p(x), _stream(stream)))
    return x


def op_embed(ctx: Context, embed: torch.Tensor, tok: torch.Tensor, stream=None):
    h = torch.empty(tok.numel(), ctx.shape.d_model, dtype=torch.float32, device=tok.device)
    check(lib().cb_op_embed(ctx.handle, _p(embed), _p(tok), tok.numel(), _p(h), _stream(stream)))
    return h


__all__ = ["Context", "Group", "nccl_unique_id", "ModelWeights", "controller_ratio", "controller_pick_device", "kv_to_paged", "Store", "chunk_digest", "model_identity",
           "blend_request_store", "CacheBlendError", "schedule", "rope_realign", "kv_deviation_topk",
           "blend_layer", "blend_forward", "gen_fill", "gen_ints", "op_gemm", "op_attention", "op_rmsnorm",
           "op_embed"]
