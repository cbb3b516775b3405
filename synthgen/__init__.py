"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no routing, no scoring,
no quantisation, no FFN).  It only draws numbers.  It is the single piece of
code both sides of the parity tests may use.

Generator (counter based, so the CUDA kernel `hb_synth_fill_f16` in
paper_2411_01433_b200/csrc/synth.cu reproduces it bit for bit):

    key          = stream_key(seed, *ids)                  (host only, 64-bit)
    u_i          = mix64(key + (i + 1) * GOLDEN  mod 2^64)  (splitmix64 finaliser)
    s_i          = sum of the four 16-bit fields of u_i  - 131070     (int, |s|<2^18)
    value_i      = fp16_rne( fp32(s_i) * c )      c = fp32(sigma / STD4)

s_i is an Irwin-Hall(4) draw: symmetric, unit-scaled by STD4 to standard
deviation sigma, bounded at +-3.46 sigma.  Every step is an exact integer op or
one IEEE fp32 multiply followed by one fp32->fp16 round-to-nearest-even, which
numpy and CUDA (`__fmul_rn`, `__float2half_rn`) perform identically.

Workload recipe:
    router  W_g[l]        ~ N(0, sigma_r^2 / H)   sigma_r = 1.5 (Mixtral) / 1.8 (Phi)
    W1, W3 of expert (l,e) ~ N(0, 1/H)
    W2 of expert (l,e)     ~ N(0, 1/F)
    x (token t, layer l)   ~ N(0, 1)
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1
# standard deviation of the sum of four independent uniforms on {0..65535}
STD4 = math.sqrt(4.0 * (65536.0 ** 2 - 1.0) / 12.0)

# stream kinds
KIND_ROUTER = 1
KIND_EXPERT = 2
KIND_X = 3
KIND_DELTA = 4

DEFAULT_SEED = 1433


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on a Python int (host-side key derivation)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def stream_key(seed: int, *ids: int) -> int:
    """64-bit key of one stream: folds the ids into the seed one at a time."""
    k = mix64_int(seed + GOLDEN)
    for i in ids:
        k = mix64_int((k ^ (int(i) & MASK64)) + GOLDEN)
    return k


def scale_f32(sigma: float) -> np.float32:
    """The fp32 multiplier c for a target standard deviation sigma."""
    return np.float32(sigma / STD4)


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def irwin_hall_int(key: int, n: int, start: int = 0) -> np.ndarray:
    """s_i for i in [start, start+n) as int32."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(key) + i * np.uint64(GOLDEN)
        u = _mix64_np(z)
    m = np.uint64(0xFFFF)
    s = ((u & m) + ((u >> np.uint64(16)) & m) + ((u >> np.uint64(32)) & m)
         + (u >> np.uint64(48)))
    return s.astype(np.int64).astype(np.int32) - np.int32(131070)


def fill_f16(key: int, n: int, sigma: float, start: int = 0) -> np.ndarray:
    """n fp16 values of stream `key` (elements start..start+n-1)."""
    out = np.empty(n, dtype=np.float16)
    c = scale_f32(sigma)
    step = 1 << 18                    # chunked so the uint64 temporaries stay in cache

    def chunk(a):
        b = min(n, a + step)
        s = irwin_hall_int(key, b - a, start + a).astype(np.float32)
        out[a:b] = (s * c).astype(np.float16)   # one IEEE fp32 multiply, then RNE

    starts = range(0, n, step)
    if n <= 4 * step:
        for a in starts:
            chunk(a)
    else:                             # numpy releases the GIL: use the host's cores
        with ThreadPoolExecutor(max_workers=min(16, len(os.sched_getaffinity(0)))) as ex:
            list(ex.map(chunk, starts))
    return out


# ---------------------------------------------------------------- workloads

class MoEShape:
    """Shape of one MoE model's expert layers."""

    def __init__(self, name, n_layers, n_experts, top_k, hidden, ffn, sigma_router):
        self.name = name
        self.n_layers = n_layers
        self.n_experts = n_experts
        self.top_k = top_k
        self.hidden = hidden
        self.ffn = ffn
        self.sigma_router = sigma_router

    def __repr__(self):
        return (f"MoEShape({self.name}: L={self.n_layers} E={self.n_experts} "
                f"k={self.top_k} H={self.hidden} F={self.ffn})")


TINY = MoEShape("tiny", 2, 8, 2, 256, 512, 1.5)
MIXTRAL = MoEShape("mixtral-8x7b", 32, 8, 2, 4096, 14336, 1.5)
PHI = MoEShape("phi-3.5-moe", 32, 16, 2, 4096, 6400, 1.8)


def router_weights(shape: MoEShape, layer: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """W_g of `layer`, fp16 [E, H] ~ N(0, sigma_r^2/H)."""
    key = stream_key(seed, KIND_ROUTER, layer)
    sig = shape.sigma_router / math.sqrt(shape.hidden)
    return fill_f16(key, shape.n_experts * shape.hidden, sig).reshape(
        shape.n_experts, shape.hidden)


def expert_key(seed: int, layer: int, expert: int, mat: int) -> int:
    return stream_key(seed, KIND_EXPERT, layer, expert, mat)


def expert_sigma(shape: MoEShape, mat: int) -> float:
    """mat 0 = W1 [F,H], 1 = W3 [F,H], 2 = W2 [H,F]."""
    return 1.0 / math.sqrt(shape.hidden if mat < 2 else shape.ffn)


def expert_weights(shape: MoEShape, layer: int, expert: int, seed: int = DEFAULT_SEED):
    """(W1 [F,H], W3 [F,H], W2 [H,F]) fp16 of expert (layer, expert)."""
    H, F = shape.hidden, shape.ffn
    out = []
    for mat, (n, k) in enumerate(((F, H), (F, H), (H, F))):
        key = expert_key(seed, layer, expert, mat)
        out.append(fill_f16(key, n * k, expert_sigma(shape, mat)).reshape(n, k))
    return tuple(out)


def hidden_states(shape: MoEShape, token: int, layer: int, batch: int = 1,
                  seed: int = DEFAULT_SEED) -> np.ndarray:
    """Gating input x for (token step, layer): fp16 [batch, H] ~ N(0,1), iid."""
    key = stream_key(seed, KIND_X, token, layer)
    return fill_f16(key, batch * shape.hidden, 1.0).reshape(batch, shape.hidden)


def correlated_states(shape: MoEShape, n_tokens: int, cos_layer: float, rho: float,
                      seed: int = DEFAULT_SEED) -> np.ndarray:
    """Gating inputs with layer-to-layer cosine ~cos_layer and token locality rho.

    Used by the constrained-cache config:
        x(t,0)   = rho*x(t-1,0) + sqrt(1-rho^2)*d
        x(t,l+1) = c*x(t,l) + sqrt(1-c^2)*d
    with d ~ N(0,1) per (t,l) from stream KIND_DELTA.  Mixing is done in fp64
    and rounded once to fp16.  Returns fp16 [n_tokens, n_layers, H].
    """
    H, L = shape.hidden, shape.n_layers
    out = np.empty((n_tokens, L, H), dtype=np.float16)
    prev0 = None
    for t in range(n_tokens):
        d = fill_f16(stream_key(seed, KIND_DELTA, t, 0), H, 1.0).astype(np.float64)
        x = d if prev0 is None else rho * prev0 + math.sqrt(1 - rho * rho) * d
        prev0 = x
        cur = x
        out[t, 0] = cur.astype(np.float16)
        for l in range(1, L):
            d = fill_f16(stream_key(seed, KIND_DELTA, t, l), H, 1.0).astype(np.float64)
            cur = cos_layer * cur + math.sqrt(1 - cos_layer * cos_layer) * d
            out[t, l] = cur.astype(np.float16)
    return out
