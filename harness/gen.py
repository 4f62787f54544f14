"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

TEST/BENCH INFRASTRUCTURE, NOT THE METHOD: nothing here computes any part of
HeteGen (no product, no partition, no cost model).  It only produces input bits.

Recipe (SURVEY.md 8(d) "Generator"):
    key   = splitmix64(seed ^ splitmix64(tensor_id))
    u_i   = (splitmix64(key + i) >> 11) * 2**-53
    value = (2*u_i - 1) * a   -> float32 (RNE) -> bf16 (RNE)
Scales: x a=sqrt(3) (unit variance); W a=sqrt(3/K) (unit-variance y); bias a=0.1.
Tensor ids: (layer << 8) | (linear << 4) | role, linear in {qkv=0,o=1,fc1=2,fc2=3},
role in {W=0, bias=1, x=2}.  Seeds: base 1164 + config index (+ decode step for x).

Two implementations: `*_np` (pure numpy, slow, the cross-check) and the ctypes
wrapper over harness/libhgen.so (multi-threaded, used for GB-sized weights).
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

BASE_SEED = 1164
LINEARS = {"qkv": 0, "o": 1, "fc1": 2, "fc2": 3}
ROLES = {"W": 0, "bias": 1, "x": 2}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def tensor_id(layer: int, linear: str | int, role: str | int) -> int:
    lin = LINEARS[linear] if isinstance(linear, str) else int(linear)
    rol = ROLES[role] if isinstance(role, str) else int(role)
    return (int(layer) << 8) | (lin << 4) | rol


def w_scale(K: int) -> float:
    return math.sqrt(3.0 / K)


X_SCALE = math.sqrt(3.0)
BIAS_SCALE = 0.1


# ---------------------------------------------------------------- numpy version
def splitmix64_np(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def key_np(seed: int, tid: int) -> np.uint64:
    return splitmix64_np(np.uint64(seed) ^ splitmix64_np(np.uint64(tid)))


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (uint16)."""
    u = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def uniform_bf16_np(seed: int, tid: int, n: int, a: float, offset: int = 0) -> np.ndarray:
    k = key_np(seed, tid)
    with np.errstate(over="ignore"):
        idx = k + np.uint64(offset) + np.arange(n, dtype=np.uint64)
    u = (splitmix64_np(idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    v = (2.0 * u - 1.0) * a
    return f32_to_bf16_bits(v.astype(np.float32))


def int_bf16_np(seed: int, tid: int, n: int, m: int, offset: int = 0) -> np.ndarray:
    k = key_np(seed, tid)
    with np.errstate(over="ignore"):
        idx = k + np.uint64(offset) + np.arange(n, dtype=np.uint64)
    u = (splitmix64_np(idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    v = np.floor(u * float(2 * m + 1)) - float(m)
    return f32_to_bf16_bits(v.astype(np.float32))


# ---------------------------------------------------------------- C version
_LIB = None
_HERE = os.path.dirname(os.path.abspath(__file__))


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libhgen.so")
        if not os.path.exists(path):
            from tools.build import build_harness  # noqa: local import, build on demand
            build_harness()
        L = ctypes.CDLL(path)
        u64, i32, dbl, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.hgen_splitmix64.restype = u64
        L.hgen_splitmix64.argtypes = [u64]
        L.hgen_uniform_bf16.argtypes = [u64, u64, u64, u64, dbl, vp, i32]
        L.hgen_int_bf16.argtypes = [u64, u64, u64, u64, i32, vp, i32]
        L.hgen_uniform_f32.argtypes = [u64, u64, u64, u64, dbl, vp, i32]
        _LIB = L
    return _LIB


def _threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def uniform_bf16(seed: int, tid: int, n: int, a: float, offset: int = 0, out=None, nthreads=None):
    """n bf16 bit patterns (uint16 ndarray, or fill `out` = any writable buffer address holder).

    `out` may be a numpy uint16 array or an integer address (e.g. a pinned torch
    tensor's data_ptr()) with room for n uint16.
    """
    if out is None:
        out = np.empty(n, dtype=np.uint16)
    addr = out if isinstance(out, int) else out.ctypes.data
    lib().hgen_uniform_bf16(seed, tid, offset, n, a, addr, nthreads or _threads())
    return out


def int_bf16(seed: int, tid: int, n: int, m: int, offset: int = 0, out=None, nthreads=None):
    if out is None:
        out = np.empty(n, dtype=np.uint16)
    addr = out if isinstance(out, int) else out.ctypes.data
    lib().hgen_int_bf16(seed, tid, offset, n, m, addr, nthreads or _threads())
    return out


# ---------------------------------------------------------------- linear inputs
def linear_inputs(seed: int, layer: int, linear: str, B: int, N: int, K: int,
                  bias: bool = True, integer: int = 0):
    """(x[B,K], W[N,K], bias[N] or None) as bf16 bit arrays (bias as float32).

    integer>0 draws small integers in [-integer, integer] (exact-arithmetic tests).
    """
    tx, tw, tb = (tensor_id(layer, linear, r) for r in ("x", "W", "bias"))
    if integer:
        x = int_bf16(seed, tx, B * K, integer).reshape(B, K)
        W = int_bf16(seed, tw, N * K, integer).reshape(N, K)
        b = bf16_bits_to_f32(int_bf16(seed, tb, N, integer)) if bias else None
    else:
        x = uniform_bf16(seed, tx, B * K, X_SCALE).reshape(B, K)
        W = uniform_bf16(seed, tw, N * K, w_scale(K)).reshape(N, K)
        b = bf16_bits_to_f32(uniform_bf16(seed, tb, N, BIAS_SCALE)) if bias else None
    return x, W, b
