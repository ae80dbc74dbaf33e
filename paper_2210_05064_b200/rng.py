"""CounterRng / splitmix64 / mix (rng.hpp:16-75) in Python.

Scalar ``CounterRng`` reproduces the reference's draws bit-for-bit (same
integer mixing; Box-Muller through the platform libm like the reference).
``normal_array``/``uniform_array`` are the vectorised forms used by the
synthetic workload generator.
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix(a: int, b: int) -> int:
    return splitmix64(a ^ ((0x9E3779B97F4A7C15 + ((b << 6) & M64) + (b >> 2) + splitmix64(b)) & M64))


class CounterRng:
    def __init__(self, seed: int | None = None, key: int | None = None):
        self.key = key if key is not None else (splitmix64(seed & M64) if seed is not None else 0)
        self.counter = 0

    def stream(self, *ids: int) -> "CounterRng":
        k = self.key
        for i in ids:
            k = mix(k, i & M64)
        return CounterRng(key=k)

    def next_u64(self) -> int:
        v = mix(self.key, self.counter)
        self.counter += 1
        return v

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform_int(self, n: int) -> int:
        return self.next_u64() % n

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 <= 0:
            u1 = 2.0 ** -53
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


# ------------------------------------------------------------- vectorised
_C1 = np.uint64(0x9E3779B97F4A7C15)
_C2 = np.uint64(0xBF58476D1CE4E5B9)
_C3 = np.uint64(0x94D049BB133111EB)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64) + _C1
        x = (x ^ (x >> np.uint64(30))) * _C2
        x = (x ^ (x >> np.uint64(27))) * _C3
        return x ^ (x >> np.uint64(31))


def mix_np(a, b) -> np.ndarray:
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64_np(a ^ (_C1 + (b << np.uint64(6)) + (b >> np.uint64(2)) + splitmix64_np(b)))


def uniform_np(key: int, counters: np.ndarray) -> np.ndarray:
    u = mix_np(np.uint64(key), counters.astype(np.uint64))
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal_np(key: int, n: int, start: int = 0) -> np.ndarray:
    """n normals of CounterRng(key) starting at counter `start` (2 draws each)."""
    c = np.arange(start, start + 2 * n, dtype=np.uint64)
    u = uniform_np(key, c).reshape(n, 2)
    u1 = np.where(u[:, 0] <= 0, 2.0 ** -53, u[:, 0])
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[:, 1])
