"""Counter-based random numbers on torch int64 tensors (CPU or CUDA).

rand_u32(seed, stream, idx) is a pure function of (seed, stream, idx): a
bijective 32-bit integer mixer (xor-shift / multiply, "lowbias32" style
constants) applied twice with stream keys. All intermediate products are split
so that no int64 multiplication ever overflows, which makes the result
bit-identical on every device and every torch build.
"""

import torch

M32 = 0xFFFFFFFF
_C1 = 0x7FEB352D
_C2 = 0x846CA68B


def _mulmod32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    xh = x >> 16
    xl = x & 0xFFFF
    return ((((xh * c) & 0xFFFF) << 16) + xl * c) & M32


def _mix32_t(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mulmod32(x, _C1)
    x = x ^ (x >> 15)
    x = _mulmod32(x, _C2)
    x = x ^ (x >> 16)
    return x


def _mix32_i(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * _C1) & M32
    x ^= x >> 15
    x = (x * _C2) & M32
    x ^= x >> 16
    return x


def _stream_keys(seed: int, stream: int):
    k1 = _mix32_i(_mix32_i(seed * 0x9E3779B1 + 0x632BE5AB) ^ (stream * 0x85EBCA77))
    k2 = _mix32_i(k1 ^ 0xC2B2AE3D ^ _mix32_i(stream + 0x27D4EB2F))
    return k1, k2


def rand_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Uniform 32-bit values (as int64 in [0, 2^32)) for counters idx (int64, < 2^32)."""
    k1, k2 = _stream_keys(seed, stream)
    x = (idx.to(torch.int64) & M32) ^ k1
    x = _mix32_t(x)
    x = x ^ k2
    return _mix32_t(x)


def rand_uniform_int(seed: int, stream: int, idx: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Uniform integers in [lo, hi] (inclusive), hi - lo < 2^31."""
    span = hi - lo + 1
    assert 0 < span < (1 << 31)
    return lo + ((rand_u32(seed, stream, idx) * span) >> 32)


def rand_unit_f64(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Uniform doubles in (0, 1) with 53 random bits (two 32-bit draws)."""
    a = rand_u32(seed, stream, idx)
    b = rand_u32(seed, stream + 0x10000, idx)
    u53 = (a << 21) | (b >> 11)
    return (u53.to(torch.float64) + 0.5) * (1.0 / float(1 << 53))
