"""Counter-based RNG spec shared (as a SPEC, not as code) by the oracle and the CUDA path.

This module holds none of CacheBlend's arithmetic. It only turns
(seed, stream, index) into numbers. The CUDA library implements the same spec
independently in `paper_2405_16444_b200/csrc/gen.cu` (`cb_gen_fill`), and
`tests/test_gpu_parity.py::test_gen_fill_bitexact` checks the two bit-for-bit on samples.

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


_CHUNK = 1 << 20  # elements per worker task (numpy releases the GIL inside these ufuncs)


def _mix_inplace(z: np.ndarray) -> None:
    """mix64 on a uint64 array, in place (same operations as `mix64`, fewer temporaries)."""
    z += _GOLDEN
    z ^= z >> np.uint64(30)
    z *= _C1
    z ^= z >> np.uint64(27)
    z *= _C2
    z ^= z >> np.uint64(31)


def _parallel(count: int, fn) -> None:
    """Runs fn(lo, hi) over [0, count) in chunks on a thread pool (results are written by index, so the
    values do not depend on the split)."""
    if count <= _CHUNK:
        if count:
            fn(0, count)
        return
    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda lo: fn(lo, min(count, lo + _CHUNK)), range(0, count, _CHUNK)))


def _raw_into(base: int, start: int, lo: int, hi: int) -> np.ndarray:
    z = np.arange(start + lo, start + hi, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z += np.uint64(base)
        _mix_inplace(z)
    return z


def raw(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    base = stream_base(seed, stream)
    out = np.empty(count, dtype=np.uint64)

    def fn(lo, hi):
        out[lo:hi] = _raw_into(base, start, lo, hi)
    _parallel(count, fn)
    return out


def _u_from_raw(z: np.ndarray) -> np.ndarray:
    k = (z >> np.uint64(40)).astype(np.float32)
    k *= np.float32(2.0 ** -23)
    k -= np.float32(1.0)
    return k


def uniform_pm1(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """u in [-1, 1) as float32, exactly k * 2**-23 - 1 with k a 24-bit integer."""
    return _u_from_raw(raw(seed, stream, start, count))


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round to nearest even. Inputs are finite."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    return ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def _values_chunk(base: int, start: int, lo: int, hi: int, scale: float, offset: float, dtype: str) -> np.ndarray:
    u = _u_from_raw(_raw_into(base, start, lo, hi))
    v = (np.float32(offset) + u * np.float32(scale)).astype(np.float32)
    if dtype == "bf16":
        return bf16_bits_to_f32(to_bf16_bits(v))
    return v


def values_f32(seed: int, stream: int, count: int, scale: float, offset: float = 0.0,
               start: int = 0) -> np.ndarray:
    """fp32(offset + fp32(u * scale)), the fp32 storage mode of the spec."""
    return values(seed, stream, count, scale, offset, "f32", start)


def values(seed: int, stream: int, count: int, scale: float, offset: float = 0.0,
           dtype: str = "bf16", start: int = 0) -> np.ndarray:
    """Values as they are stored for `dtype` ('bf16' or 'f32'), returned as float32 arrays
    (bf16 values are exactly representable in float32)."""
    if dtype not in ("bf16", "f32"):
        raise ValueError(f"unknown dtype {dtype!r}")
    base = stream_base(seed, stream)
    out = np.empty(count, dtype=np.float32)

    def fn(lo, hi):
        out[lo:hi] = _values_chunk(base, start, lo, hi, scale, offset, dtype)
    _parallel(count, fn)
    return out


def ints(seed: int, stream: int, count: int, modulus: int, start: int = 0) -> np.ndarray:
    r = raw(seed, stream, start, count)
    return (r % np.uint64(modulus)).astype(np.int64)
