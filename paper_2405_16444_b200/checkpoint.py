"""Loading a Llama/Mistral-family checkpoint in the Hugging Face safetensors layout.

The paper runs CacheBlend on Mistral-7B, Yi-34B and Llama-70B checkpoints and hands the fused
KV cache to the serving engine. This module reads such a checkpoint into the C-ABI weight layout
(include/cacheblend.h cb_layer_w) without any method arithmetic:

  * safetensors: an 8-byte little-endian header length, a JSON header {name: {dtype, shape, data_offsets}},
    then the raw little-endian tensor bytes; read through mmap, one layer at a time, so host memory holds
    at most one layer's tensors. Sharded checkpoints list their files in model.safetensors.index.json.
  * config.json -> ModelShape (hidden_size, num_hidden_layers, num_attention_heads, num_key_value_heads,
    head_dim, intermediate_size, vocab_size, rope_theta, rms_norm_eps).
  * q_proj / k_proj / v_proj are stacked into w_qkv (q heads, k heads, v heads) and gate_proj / up_proj
    into w_gate_up (gate rows, then up rows); o_proj and down_proj are already [out][in].
  * These checkpoints rotate half-split RoPE pairs (i, i + hd/2); the library rotates interleaved pairs
    (P:2531-2538). The q and k rows are permuted per head at load time (dist.interleave_rope_weights,
    DESIGN.md R9), and a K cache produced by a half-split engine goes through `engine_k_to_library` before
    the blend and `library_k_to_engine` after it (V is unaffected).

There is no fallback: a missing tensor or a shape that disagrees with config.json raises.
"""
from __future__ import annotations

import json
import mmap
import os
import struct
import warnings
from typing import Dict, Iterator, List, Optional, Tuple

import numpy as np
import torch

from . import dist as D
from .api import TORCH_DTYPES, ModelWeights

_ST_DTYPES = {"BF16": torch.bfloat16, "F16": torch.float16, "F32": torch.float32, "F64": torch.float64}


class SafetensorsFile:
    """One .safetensors file, memory-mapped; `tensor(name)` returns a CPU tensor viewing the mapping."""

    def __init__(self, path: str):
        self.path = path
        self._f = open(path, "rb")
        self._mm = mmap.mmap(self._f.fileno(), 0, access=mmap.ACCESS_READ)
        if len(self._mm) < 8:
            raise ValueError(f"{path}: not a safetensors file (shorter than its header length)")
        (n,) = struct.unpack("<Q", self._mm[:8])
        if 8 + n > len(self._mm):
            raise ValueError(f"{path}: header length {n} exceeds the file size {len(self._mm)}")
        header = json.loads(bytes(self._mm[8:8 + n]).decode("utf-8"))
        header.pop("__metadata__", None)
        self.base = 8 + n
        self.entries: Dict[str, Tuple[str, List[int], int, int]] = {}
        for name, e in header.items():
            b0, b1 = e["data_offsets"]
            if not (0 <= b0 <= b1 <= len(self._mm) - self.base):
                raise ValueError(f"{path}: tensor {name} has data_offsets {b0}..{b1} outside the file")
            self.entries[name] = (e["dtype"], list(e["shape"]), b0, b1)

    def names(self) -> List[str]:
        return list(self.entries)

    def tensor(self, name: str) -> torch.Tensor:
        dt, shape, b0, b1 = self.entries[name]
        if dt not in _ST_DTYPES:
            raise ValueError(f"{self.path}: tensor {name} has unsupported dtype {dt}")
        td = _ST_DTYPES[dt]
        count = int(np.prod(shape)) if shape else 1
        if (b1 - b0) != count * torch.empty(0, dtype=td).element_size():
            raise ValueError(f"{self.path}: tensor {name}: {b1 - b0} bytes for shape {shape} of {dt}")
        if count == 0:
            return torch.empty(shape, dtype=td)
        buf = memoryview(self._mm)[self.base + b0:self.base + b1]
        with warnings.catch_warnings():  # read-only mapping: the loader copies before anything could write
            warnings.simplefilter("ignore", UserWarning)
            return torch.frombuffer(buf, dtype=td).reshape(shape)

    def close(self):
        try:
            self._mm.close()
        except BufferError:  # a returned view is still alive; the mapping goes with it
            pass
        self._f.close()


class Checkpoint:
    """A checkpoint directory: config.json plus model.safetensors or model.safetensors.index.json + shards."""

    def __init__(self, directory: str):
        self.dir = directory
        with open(os.path.join(directory, "config.json")) as f:
            self.config = json.load(f)
        idx = os.path.join(directory, "model.safetensors.index.json")
        self.files: Dict[str, SafetensorsFile] = {}
        self.where: Dict[str, str] = {}
        if os.path.exists(idx):
            with open(idx) as f:
                self.where = dict(json.load(f)["weight_map"])
        else:
            single = os.path.join(directory, "model.safetensors")
            if not os.path.exists(single):
                raise FileNotFoundError(f"{directory}: neither model.safetensors nor model.safetensors.index.json")
            self.where = {n: "model.safetensors" for n in self._file("model.safetensors").names()}

    def _file(self, fname: str) -> SafetensorsFile:
        if fname not in self.files:
            self.files[fname] = SafetensorsFile(os.path.join(self.dir, fname))
        return self.files[fname]

    def tensor(self, name: str) -> torch.Tensor:
        if name not in self.where:
            raise KeyError(f"{self.dir}: checkpoint has no tensor {name}")
        return self._file(self.where[name]).tensor(name)

    def close(self):
        for f in self.files.values():
            f.close()
        self.files.clear()


def shape_from_config(config: Dict, name: Optional[str] = None, max_context: Optional[int] = None):
    """config.json of a Llama/Mistral-family model -> synth.workload.ModelShape. Raises for what the kernels
    do not compute: another activation, scaled RoPE, or a sliding attention window shorter than
    `max_context` (the longest blended request; the kernels attend over the whole causal prefix)."""
    from synth.workload import ModelShape
    d, nq = int(config["hidden_size"]), int(config["num_attention_heads"])
    hd = config.get("head_dim") or d // nq
    if config.get("hidden_act", "silu") != "silu":
        raise ValueError(f"unsupported hidden_act {config.get('hidden_act')} (the block is SwiGLU, R-model)")
    rp = config.get("rope_parameters") or {}  # newer config.json files; older ones carry rope_theta/rope_scaling
    if config.get("rope_scaling") or rp.get("rope_type", "default") != "default":
        raise ValueError("scaled RoPE is not supported (plain RoPE theta_i = theta^(-2i/hd), R8)")
    theta = float(rp.get("rope_theta", config.get("rope_theta", 10000.0)))
    win = config.get("sliding_window")
    if win is not None and (max_context is None or max_context > int(win)):
        raise ValueError(f"sliding_window {win}: pass max_context <= {win} (the kernels attend over the whole "
                         "causal prefix)")
    return ModelShape(name or config.get("model_type", "hf"), int(config["num_hidden_layers"]), d, nq,
                      int(config.get("num_key_value_heads", nq)), int(hd), int(config["intermediate_size"]),
                      int(config["vocab_size"]), theta, float(config.get("rms_norm_eps", 1e-5)))


def _expect(t: torch.Tensor, shape, name: str) -> torch.Tensor:
    if list(t.shape) != list(shape):
        raise ValueError(f"tensor {name} has shape {list(t.shape)}, config.json implies {list(shape)}")
    return t


def iter_layers(ck: Checkpoint, shape, dtype: str, device, rope: str = "half") -> Iterator[Dict[str, torch.Tensor]]:
    """Yield each layer's weights in the cb_layer_w layout on `device` (one layer in host memory at a time)."""
    td = TORCH_DTYPES[dtype]
    s = shape
    for i in range(s.n_layers):
        p = f"model.layers.{i}."
        g = lambda n, shp: _expect(ck.tensor(p + n), shp, p + n)
        qkv = torch.cat([g("self_attn.q_proj.weight", [s.qd, s.d_model]),
                         g("self_attn.k_proj.weight", [s.kvd, s.d_model]),
                         g("self_attn.v_proj.weight", [s.kvd, s.d_model])], 0)
        if rope == "half":
            qkv = D.interleave_rope_weights(qkv, s)
        elif rope != "interleaved":
            raise ValueError(f"rope must be 'half' or 'interleaved', not {rope!r}")
        up = lambda t, dt=td: t.to(device=device, dtype=dt, copy=True).contiguous()  # never a view of the mmap
        yield {"attn_norm": up(g("input_layernorm.weight", [s.d_model]), torch.float32),
               "w_qkv": up(qkv),
               "w_o": up(g("self_attn.o_proj.weight", [s.d_model, s.qd])),
               "mlp_norm": up(g("post_attention_layernorm.weight", [s.d_model]), torch.float32),
               "w_gate_up": up(torch.cat([g("mlp.gate_proj.weight", [s.d_ff, s.d_model]),
                                          g("mlp.up_proj.weight", [s.d_ff, s.d_model])], 0)),
               "w_down": up(g("mlp.down_proj.weight", [s.d_model, s.d_ff]))}


def load(directory: str, dtype: str = "bf16", device="cuda", rope: str = "half", max_context: Optional[int] = None):
    """Read a Hugging Face Llama/Mistral checkpoint -> (ModelShape, ModelWeights on `device`).
    rope='half' (Hugging Face convention) permutes q/k rows to the library's interleaved pairs."""
    ck = Checkpoint(directory)
    try:
        s = shape_from_config(ck.config, max_context=max_context)
        embed = _expect(ck.tensor("model.embed_tokens.weight"), [s.vocab, s.d_model], "model.embed_tokens.weight")
        embed = embed.to(device=device, dtype=TORCH_DTYPES[dtype], copy=True).contiguous()
        layers = list(iter_layers(ck, s, dtype, device, rope))
    finally:
        ck.close()
    return s, ModelWeights(s, dtype, embed, layers)


def engine_k_to_library(k: torch.Tensor) -> torch.Tensor:
    """A half-split engine's cached K [..., head_dim] -> the library's interleaved order."""
    return D.interleave_rope_cache(k)


def library_k_to_engine(k: torch.Tensor) -> torch.Tensor:
    """The blended K back to the half-split engine's order."""
    return D.interleave_rope_cache(k, inverse=True)
