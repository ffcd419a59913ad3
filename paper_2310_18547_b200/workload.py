"""Batch-composition generators of the reference (workload.hpp / workload.cpp),
host-side, used to lay out synthetic SGMV segments the way the reference does.

* ``Rng`` -- mt19937_64 with the reference's hand-rolled distributions
  (workload.hpp:13-42, workload.cpp:11-36);
* ``derive_seed`` (workload.cpp:38-44), ``model_count_for`` (:92-104),
  ``assign_models`` (:106-143): per-request adapter ids under the paper's
  Distinct / Uniform / Skewed / Identical popularity;
* ``group_segments``: rows grouped by ascending adapter id, the layout
  verify_sgmv builds (experiments.cpp:56-76).

Pinned against the reference's golden draws in tests/golden/rng.json
(tests/test_workload.py).
"""
from __future__ import annotations

import math

DISTINCT, UNIFORM, SKEWED, IDENTICAL = 0, 1, 2, 3
_M64 = (1 << 64) - 1


class Rng:
    _N, _M = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self._N
        mt[0] = seed & _M64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt, self._i = mt, self._N

    def _twist(self):
        mt, n, m = self._mt, self._N, self._M
        for i in range(n):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % n] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + m) % n] ^ xa
        self._i = 0

    def next(self) -> int:
        if self._i >= self._N:
            self._twist()
        x = self._mt[self._i]
        self._i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64

    def uniform01(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def uniform_index(self, n: int) -> int:
        if n <= 0:
            raise ValueError("Rng::uniform_index: n must be > 0")
        limit = _M64 - _M64 % n
        while True:
            x = self.next()
            if x < limit:
                return x % n

    def uniform_int(self, lo: int, hi: int) -> int:
        if hi < lo:
            raise ValueError("Rng::uniform_int: empty range")
        return lo + self.uniform_index(hi - lo + 1)

    def discrete(self, cumulative, total: float) -> int:
        u = self.uniform01() * total
        lo, hi = 0, len(cumulative)
        while lo < hi:  # std::upper_bound
            mid = (lo + hi) // 2
            if u < cumulative[mid]:
                hi = mid
            else:
                lo = mid + 1
        return len(cumulative) - 1 if lo == len(cumulative) else lo

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.uniform_index(i)
            v[i - 1], v[j] = v[j], v[i - 1]


def derive_seed(seed: int, stream: int) -> int:
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def model_count_for(n: int, popularity: int) -> int:
    if n <= 0:
        return 0
    if popularity == DISTINCT:
        return n
    if popularity == IDENTICAL:
        return 1
    return int(math.ceil(math.sqrt(float(n))))


def assign_models(n: int, popularity: int, alpha: float, seed: int) -> list:
    if n < 0:
        raise ValueError("assign_models: negative request count")
    out = [0] * n
    if n == 0:
        return out
    rng = Rng(seed)
    if popularity == DISTINCT:
        out = list(range(n))
    elif popularity == UNIFORM:
        m = model_count_for(n, popularity)
        out = [i % m for i in range(n)]
        rng.shuffle(out)
    elif popularity == SKEWED:
        if alpha <= 1.0:
            raise ValueError("assign_models: Skewed needs alpha > 1")
        m = model_count_for(n, popularity)
        cumulative, total, w = [], 0.0, 1.0
        for _ in range(m):
            total += w
            cumulative.append(total)
            w /= alpha
        out = [rng.discrete(cumulative, total) for _ in range(n)]
    return out


def group_segments(ids: list):
    """Rows grouped by ascending adapter id, original order within (experiments.cpp:56-76).

    Returns (bounds [n+1], adapter ids [n], row order [s_n] = gathered row -> original row).
    """
    uniq = sorted(set(ids))
    order = sorted(range(len(ids)), key=lambda i: (ids[i], i))
    bounds = [0]
    for u in uniq:
        bounds.append(bounds[-1] + sum(1 for i in ids if i == u))
    return bounds, uniq, order
