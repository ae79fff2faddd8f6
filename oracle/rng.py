"""Bit-exact Python restatement of the reference's seeded generator
(proj/include/fsk/rng.hpp:12-99): xoshiro256** seeded through splitmix64,
Box-Muller normals with a fixed consumption order, Dirichlet(1..1) simplex
weights. Test infrastructure (small sizes); the product carries its own C++
implementation (include/fsk/rng.hpp) for bulk synthetic inputs.
"""
from __future__ import annotations

import math

import numpy as np

_M = (1 << 64) - 1


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & _M


class Rng:
    def __init__(self, seed: int):
        x = seed & _M
        s = []
        for _ in range(4):  # splitmix64, rng.hpp:16-23
            x = (x + 0x9E3779B97F4A7C15) & _M
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
            s.append(z ^ (z >> 31))
        self.s = s
        self.has_spare = False
        self.spare = 0.0

    def next_u64(self) -> int:  # rng.hpp:27-37
        s = self.s
        result = (_rotl((s[1] * 5) & _M, 7) * 9) & _M
        t = (s[1] << 17) & _M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def uniform(self) -> float:  # rng.hpp:40
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def normal(self) -> float:  # rng.hpp:44-57
        if self.has_spare:
            self.has_spare = False
            return self.spare
        u1 = self.uniform()
        u2 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        rad = math.sqrt(-2.0 * math.log(u1))
        ang = 2.0 * math.pi * u2
        self.spare = rad * math.sin(ang)
        self.has_spare = True
        return rad * math.cos(ang)

    def normal_vector(self, n: int) -> np.ndarray:
        return np.array([self.normal() for _ in range(n)])

    def simplex_weights(self, n: int) -> np.ndarray:  # rng.hpp:67-78
        w = []
        total = 0.0
        for _ in range(n):
            u = self.uniform()
            while u <= 0.0:
                u = self.uniform()
            v = -math.log(u)
            total += v
            w.append(v)
        return np.array([v / total for v in w])


def random_measure(rng: Rng, n: int, d: int, uniform: bool = True):
    """test_stream.cpp:15-23: points row-major from rng.normal(), then weights."""
    pts = np.array([[rng.normal() for _ in range(d)] for _ in range(n)]).reshape(n, d)
    w = np.full(n, 1.0 / n) if uniform else rng.simplex_weights(n)
    return pts, w
