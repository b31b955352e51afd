"""Counter-based RNG spec shared (as a SPEC, not as code) by the oracle and the CUDA path.

This module holds none of CacheBlend's arithmetic. It only turns
(seed, stream, index) into numbers. The CUDA library implements the same spec
independently in `paper_2405_16444_b200/csrc/gen.cu` (`cb_gen_fill`), and
`tests/test_gen_parity.py` checks the two bit-for-bit on samples.

Spec (all integer arithmetic modulo 2**64):

    mix64(z)   : z += 0x9E3779B97F4A7C15
                 z  = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                 z  = (z ^ (z >> 27)) * 0x94D049BB133111EB
                 return z ^ (z >> 31)                    (splitmix64 finaliser)
    base(s, t) = mix64(mix64(seed) ^ stream)
    raw(i)     = mix64(base + i)
    u(i)       = fp32(raw(i) >> 40) * 2**-23 - 1         exact in fp32, u in [-1, 1)
    value(i)   = fp32(offset + fp32(u(i) * scale))       each op rounded to fp32 (no FMA)
    bf16 mode  : value rounded to bfloat16, round-to-nearest-even
    int mode   : raw(i) % modulus                        (token ids)
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def mix64_int(z: int) -> int:
    """Scalar splitmix64 finaliser on Python ints (reference for the vector form)."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix64(z: np.ndarray) -> np.ndarray:
    """Vector splitmix64 finaliser; uint64 numpy arithmetic wraps modulo 2**64."""
    z = z + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def stream_base(seed: int, stream: int) -> int:
    return mix64_int(mix64_int(seed & M64) ^ (stream & M64))


def raw(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    base = np.uint64(stream_base(seed, stream))
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(base + idx)


def uniform_pm1(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """u in [-1, 1) as float32, exactly k * 2**-23 - 1 with k a 24-bit integer."""
    r = raw(seed, stream, start, count)
    k = (r >> np.uint64(40)).astype(np.float32)
    return (k * np.float32(2.0 ** -23)) - np.float32(1.0)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round to nearest even. Inputs are finite."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    return ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def values_f32(seed: int, stream: int, count: int, scale: float, offset: float = 0.0,
               start: int = 0) -> np.ndarray:
    """fp32(offset + fp32(u * scale)), the fp32 storage mode of the spec."""
    u = uniform_pm1(seed, stream, start, count)
    v = u * np.float32(scale)
    return (np.float32(offset) + v).astype(np.float32)


def values(seed: int, stream: int, count: int, scale: float, offset: float = 0.0,
           dtype: str = "bf16", start: int = 0) -> np.ndarray:
    """Values as they are stored for `dtype` ('bf16' or 'f32'), returned as float32 arrays
    (bf16 values are exactly representable in float32)."""
    v = values_f32(seed, stream, count, scale, offset, start)
    if dtype == "bf16":
        return bf16_bits_to_f32(to_bf16_bits(v))
    if dtype == "f32":
        return v
    raise ValueError(f"unknown dtype {dtype!r}")


def ints(seed: int, stream: int, count: int, modulus: int, start: int = 0) -> np.ndarray:
    r = raw(seed, stream, start, count)
    return (r % np.uint64(modulus)).astype(np.int64)
