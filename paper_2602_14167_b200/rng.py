"""RngStream: the reference's counter-based SplitMix-style generator
(include/qforge/rng.hpp:12-85), restated so that parameter sets and random
Pauli sums are bit-identical to the reference's inputs.

Pinned against the reference header itself (oracle/ref_rng_driver.cpp ->
tests/golden/rng_known_answers.txt).
"""
from __future__ import annotations

import math

_M64 = (1 << 64) - 1


def _mix(z: int) -> int:  # rng.hpp:71-75
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class RngStream:
    """Output depends only on (seed, stream, counter) (rng.hpp:9-11)."""

    __slots__ = ("_seed", "_stream", "_counter", "_have_spare", "_spare", "_key")

    def __init__(self, seed: int = 0, stream: int = 0):
        self._seed = seed & _M64
        self._stream = stream & _M64
        self._counter = 0
        self._have_spare = False
        self._spare = 0.0
        # key_(), rng.hpp:76-78
        self._key = _mix(self._seed ^ 0xA0761D6478BD642F) ^ _mix(self._stream ^ 0xE7037ED1A0B428DB)

    def seed(self) -> int:
        return self._seed

    def stream(self) -> int:
        return self._stream

    def next_u64(self) -> int:  # rng.hpp:21-27
        z = (self._key + self._counter * 0x9E3779B97F4A7C15) & _M64
        self._counter += 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:  # rng.hpp:30-32
        return float(self.next_u64() >> 11) * (2.0 ** -53)

    def uniform_below(self, bound: int) -> int:  # rng.hpp:35-41
        if bound <= 1:
            return 0
        limit = _M64 - (_M64 % bound)
        while True:
            v = self.next_u64()
            if v < limit:
                return v % bound

    def normal(self) -> float:  # rng.hpp:44-57 (Box-Muller, cached spare)
        if self._have_spare:
            self._have_spare = False
            return self._spare
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 < 1e-300:
            u1 = 1e-300
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self._spare = r * math.sin(a)
        self._have_spare = True
        return r * math.cos(a)

    def split(self, n: int) -> list["RngStream"]:  # rng.hpp:60-68
        return [RngStream(self._seed, _mix(self._stream ^ _mix((0xD1B54A32D192ED03 + i) & _M64)))
                for i in range(n)]
