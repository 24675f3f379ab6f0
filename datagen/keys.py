"""Join-key generators: Zipf(s=1) on a bounded support, uniform keys, small random tables.

Zipf ranks use the rejection-inversion sampler of Hoermann & Derflinger (1996),
specialised to exponent s = 1 (h(x) = 1/x, H(x) = log x, H^-1(y) = exp y), which
is valid for s = 1 on a finite support [1, N] where numpy's zipf (s > 1) is not
(BASELINE.json configs[3] "Zipf-skewed keys (s=1.0)").
Each rejection round draws from its own counter stream, so the output is a pure
function of (seed, stream, row).
"""

import math

import torch

from .rng import rand_unit_f64, rand_uniform_int


def zipf_ranks(n: int, N: int, seed: int, stream: int = 100, device="cpu") -> torch.Tensor:
    """n samples of Zipf(s=1) ranks in [1, N] (int64)."""
    dev = torch.device(device)
    h_x1 = math.log(1.5) - 1.0
    h_n = math.log(N + 0.5)
    s_thr = 2.0 - math.exp(math.log(2.5) - 0.5)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    pending = torch.arange(n, dtype=torch.int64, device=dev)
    rnd = 0
    while pending.numel() > 0:
        u01 = rand_unit_f64(seed, stream + 2 * rnd * 0x20000, pending)
        u = h_n + u01 * (h_x1 - h_n)
        x = torch.exp(u)
        k = torch.floor(x + 0.5).clamp_(1, N)
        accept = ((k - x) <= s_thr) | (u >= torch.log(k + 0.5) - 1.0 / k)
        out[pending[accept]] = k[accept].to(torch.int64)
        pending = pending[~accept]
        rnd += 1
        if rnd > 64:  # astronomically unlikely; keep the generator total
            out[pending] = 1
            break
    return out


def zipf_keys(n: int, N: int, seed: int, stream: int = 100, device="cpu") -> torch.Tensor:
    """Zipf(s=1) keys in [0, N): key = rank - 1."""
    return zipf_ranks(n, N, seed, stream, device) - 1


def uniform_keys(n: int, N: int, seed: int, stream: int = 200, device="cpu") -> torch.Tensor:
    """Uniform keys in [0, N)."""
    idx = torch.arange(n, dtype=torch.int64, device=torch.device(device))
    return rand_uniform_int(seed, stream, idx, 0, N - 1)


def random_small_keys(n: int, lo: int, hi: int, seed: int, stream: int = 300, device="cpu",
                      dtype=torch.int64) -> torch.Tensor:
    """Uniform keys in [lo, hi] for small adversarial test tables."""
    idx = torch.arange(n, dtype=torch.int64, device=torch.device(device))
    span = hi - lo + 1
    if span < (1 << 31):
        v = rand_uniform_int(seed, stream, idx, lo, hi)
    else:  # wide spans: combine two draws (64 random bits), then reduce
        from .rng import rand_u32
        a = rand_u32(seed, stream, idx)
        b = rand_u32(seed, stream + 1, idx)
        v64 = (a << 32) | b                      # wraps into the int64 range
        if lo == -(1 << 63) and hi == (1 << 63) - 1:
            v = v64
        else:
            v = lo + torch.remainder(v64, span)
    return v.to(dtype)
