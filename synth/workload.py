"""Seeded synthetic workloads: model shapes, weight/token/cache streams, chunk layouts.

Shapes and recipes only -- no CacheBlend arithmetic lives here (no RoPE, no norm,
no attention, no selection). Both the oracle (`oracle/`) and the CUDA path draw
their inputs from this module: the oracle through the numpy generator
(`synth.counter_rng`), the CUDA path either by uploading these arrays or by
running the library's own implementation of the same counter RNG spec
(`cb_gen_fill`), which `tests/test_gpu_parity.py::test_gen_fill_bitexact` pins bit-for-bit.

Model shapes come from the public model configs (PAPER.md names the models at
P:1819 but not their shapes). Random-init recipe
(SURVEY.md §8(c) "Model"):
  linear weights  u * 1/sqrt(fan_in)         (u uniform in [-1, 1))
  norm gains      1 + 0.1 u                  (jittered so a dropped gain is caught)
  embedding       u
  chunk caches    u (random-cache mode, full-size sampled checks only); otherwise
                  they are produced by a standalone prefill of each chunk.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import counter_rng as rng

GAIN_JITTER = 0.1


@dataclasses.dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5

    @property
    def qd(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def kvd(self) -> int:
        return self.n_kv_heads * self.head_dim

    def layer_params(self) -> int:
        d = self.d_model
        return (2 * d + d * (self.qd + 2 * self.kvd) + self.qd * d + 3 * d * self.d_ff)


MODELS: Dict[str, ModelShape] = {
    # BASELINE.json configs[0]: 2 layers, 4 heads, d_model 64 (ff/vocab proposed in SURVEY §8(c)).
    "tiny": ModelShape("tiny", 2, 64, 4, 4, 16, 256, 512),
    # Test-only shape that spans several GEMM/attention tiles with hd=128 and GQA group 4.
    "small": ModelShape("small", 4, 1024, 8, 2, 128, 2816, 1000),
    "mistral-7b": ModelShape("mistral-7b", 32, 4096, 32, 8, 128, 14336, 32000),
    "yi-34b": ModelShape("yi-34b", 60, 7168, 56, 8, 128, 20480, 64000),
    "llama-70b": ModelShape("llama-70b", 80, 8192, 64, 8, 128, 28672, 32000),
}

# ---- stream ids ---------------------------------------------------------------------------
# Per-layer tensors: ((layer + 1) << 8) | code.  Global tensors: small constants below 0x100.
_CODES = {"attn_norm": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "mlp_norm": 6,
          "wg": 7, "wu": 8, "wd": 9}
STREAM_EMBED = 0xE1
STREAM_TOKENS = 0x70
STREAM_CACHE_K = 1 << 24
STREAM_CACHE_V = 2 << 24


def weight_stream(layer: int, name: str) -> int:
    return ((layer + 1) << 8) | _CODES[name]


def cache_stream(layer: int, kind: str) -> int:
    return (STREAM_CACHE_K if kind == "k" else STREAM_CACHE_V) | layer


@dataclasses.dataclass(frozen=True)
class TensorRecipe:
    """One logical tensor = `count` consecutive counter-RNG values of one stream."""
    stream: int
    shape: tuple
    scale: float
    offset: float = 0.0

    @property
    def count(self) -> int:
        return int(np.prod(self.shape))


def fp32_scale(fan_in: int) -> float:
    """The fp32 scale both generators use (the value is computed once, here)."""
    return float(np.float32(1.0 / math.sqrt(fan_in)))


def layer_recipes(m: ModelShape, layer: int) -> Dict[str, TensorRecipe]:
    d, qd, kvd, ff = m.d_model, m.qd, m.kvd, m.d_ff
    s = lambda n: weight_stream(layer, n)
    return {
        "attn_norm": TensorRecipe(s("attn_norm"), (d,), GAIN_JITTER, 1.0),
        "wq": TensorRecipe(s("wq"), (qd, d), fp32_scale(d)),
        "wk": TensorRecipe(s("wk"), (kvd, d), fp32_scale(d)),
        "wv": TensorRecipe(s("wv"), (kvd, d), fp32_scale(d)),
        "wo": TensorRecipe(s("wo"), (d, qd), fp32_scale(qd)),
        "mlp_norm": TensorRecipe(s("mlp_norm"), (d,), GAIN_JITTER, 1.0),
        "wg": TensorRecipe(s("wg"), (ff, d), fp32_scale(d)),
        "wu": TensorRecipe(s("wu"), (ff, d), fp32_scale(d)),
        "wd": TensorRecipe(s("wd"), (d, ff), fp32_scale(ff)),
    }


def embed_recipe(m: ModelShape) -> TensorRecipe:
    return TensorRecipe(STREAM_EMBED, (m.vocab, m.d_model), 1.0)


def materialize(rec: TensorRecipe, seed: int, dtype: str) -> np.ndarray:
    """Host (numpy) materialisation as float32 values exactly equal to the stored ones.
    Norm gains are always stored as fp32 (they are [d] vectors)."""
    return rng.values(seed, rec.stream, rec.count, rec.scale, rec.offset, dtype).reshape(rec.shape)


def layer_weights(m: ModelShape, layer: int, seed: int, dtype: str) -> Dict[str, np.ndarray]:
    out = {}
    for k, rec in layer_recipes(m, layer).items():
        out[k] = materialize(rec, seed, "f32" if k.endswith("norm") else dtype)
    return out


def embed_weights(m: ModelShape, seed: int, dtype: str) -> np.ndarray:
    return materialize(embed_recipe(m), seed, dtype)


# ---- requests -----------------------------------------------------------------------------
@dataclasses.dataclass
class Request:
    """One RAG-shaped blend request: context chunks (+ optional uncached suffix)."""
    chunk_lens: List[int]
    n_suffix: int
    seed: int
    ratio: float
    pos_offset: int = 0

    @property
    def n_ctx(self) -> int:
        return int(sum(self.chunk_lens))

    @property
    def n_total(self) -> int:
        return self.n_ctx + self.n_suffix

    def chunk_starts(self) -> np.ndarray:
        """Host array [n_chunks + 1]: chunk c occupies rows chunk_start[c]..chunk_start[c+1]."""
        return np.concatenate([[0], np.cumsum(self.chunk_lens)]).astype(np.int32)

    def tokens(self, vocab: int) -> np.ndarray:
        return rng.ints(self.seed, STREAM_TOKENS, self.n_total, vocab).astype(np.int32)

    def global_positions(self) -> np.ndarray:
        """g: strictly increasing global positions, default pos_offset + 0..T-1."""
        return (self.pos_offset + np.arange(self.n_total)).astype(np.int32)

    def local_positions(self) -> np.ndarray:
        """l: index of each context token within its chunk (the chunk-local RoPE position)."""
        st = self.chunk_starts()
        loc = np.zeros(self.n_ctx, dtype=np.int32)
        for c in range(len(self.chunk_lens)):
            loc[st[c]:st[c + 1]] = np.arange(st[c + 1] - st[c])
        return loc


def random_cache(m: ModelShape, layer: int, n_tok: int, seed: int, dtype: str, kind: str) -> np.ndarray:
    """Random-cache mode: cached K (already rotated at local positions) / V rows of one layer."""
    return rng.values(seed, cache_stream(layer, kind), n_tok * m.kvd, 1.0, 0.0, dtype).reshape(
        n_tok, m.n_kv_heads, m.head_dim)


STREAM_PERM = 0x5E1


def random_order(seed: int, stream: int, n: int) -> np.ndarray:
    """A seeded permutation of 0..n-1 (argsort of counter-RNG keys, ties by index)."""
    keys = rng.raw(seed, stream, 0, n)
    return np.argsort(keys, kind="stable").astype(np.int64)


def nested_selection(seed: int, n_ctx: int, k_sched: Sequence[int]) -> List[np.ndarray]:
    """Seeded replay selections S_1 >= S_2 >= ... for forced-selection runs (k_sched[i] = |S_i|, i >= 1):
    S_i = the first k_i tokens of one seeded permutation, sorted; nested because k_i is non-increasing.
    Entry 0 is all context tokens. An input recipe only (no deviation, no top-k)."""
    order = random_order(seed, STREAM_PERM, n_ctx)
    out = [np.arange(n_ctx, dtype=np.int64)]
    for k in list(k_sched)[1:]:
        out.append(np.sort(order[:int(k)]))
    return out


def sample_rows(seed: int, stream: int, n: int, k: int) -> np.ndarray:
    """k distinct seeded rows of 0..n-1, sorted."""
    return np.sort(random_order(seed, stream, n)[:min(k, n)])


# BASELINE.json configs, as concrete requests.
def config_requests(name: str, seed: int = 1) -> List[Request]:
    if name == "tiny":
        return [Request([32, 32, 32], 0, seed, 0.15)]
    if name == "mistral":
        return [Request([512] * 6, 0, seed, 0.15)]
    if name == "yi":
        return [Request([1024] * 8, 0, seed, 0.15)]
    if name == "llama":
        return [Request([1024] * 10, 0, seed, 0.15)]
    if name == "batched":
        reqs = []
        for q in range(64):
            s = seed * 1000 + q
            n_chunks = 4 + int(rng.ints(s, 0x51, 1, 5)[0])
            lens = (256 + rng.ints(s, 0x52, n_chunks, 769)).astype(int).tolist()
            reqs.append(Request(lens, 0, s, 0.15))
        return reqs
    raise ValueError(name)
