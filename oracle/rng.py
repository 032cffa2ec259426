"""ORACLE (test infrastructure only) -- CPU restatement of the reference RNG.

Restates `proj/include/cpstream/rng.hpp` of the reference:
  * SplitMix64 finalizer `mix`            (rng.hpp:14-19)
  * `derive(master, path)`                (rng.hpp:23-29)
  * frozen key kinds                      (rng.hpp:33-45)
  * `Substream`: std::mt19937_64 with 53-bit uniforms (rng.hpp:56),
    Box-Muller normals with a cached spare (rng.hpp:59-72) and column-major
    `fill_uniform` (rng.hpp:75-79).

std::mt19937_64 is not in numpy (numpy's MT19937 is the 32-bit engine), so the
engine is restated from its published definition (Matsumoto & Nishimura 2000,
C++11 [rand.predef]: w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29
d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43
f=6364136223846793005).  The twist is vectorised in three dependency-free
chunks.  Pinned by the C++ standard's known answer: the 10000th output of a
default-constructed (seed 5489) std::mt19937_64 is 9981545732273789042
([rand.predef]/4); see tests/test_oracle_kat.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1

# rng.hpp:33-45 -- frozen key kinds
K_NONTEMPORAL_SHARED = 1
K_NONTEMPORAL_PRIVATE = 2
K_TEMPORAL_SHARED = 3
K_TEMPORAL_PRIVATE = 4
K_ALS_RESTART = 5
K_ALS_FACTOR = 6
K_ALS_RESCUE = 7
K_STREAM_ALS = 8
K_SYNTH_FACTOR = 9
K_SYNTH_NOISE = 10
K_ALS_GEVD = 11


def mix(z: int) -> int:
    """rng.hpp:14-19 SplitMix64 finalizer."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def derive(master: int, path) -> int:
    """rng.hpp:23-29."""
    z = mix(master & M64)
    for k in path:
        z = mix(z ^ mix(k & M64))
    return z


_N, _M = 312, 156
_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class MT19937_64:
    """std::mt19937_64 (restated from its published definition)."""

    def __init__(self, seed: int):
        mt = [0] * _N
        mt[0] = seed & M64
        for i in range(1, _N):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & M64
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = _N
        self._buf = None

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)
        # chunk 1: i in [0,156) -- reads old mt[i+1], old mt[i+156]
        i = np.arange(0, _M)
        x = (mt[i] & _UM) | (mt[i + 1] & _LM)
        xa = (x >> one) ^ np.where((x & one) != 0, _A, np.uint64(0))
        new1 = mt[i + _M] ^ xa
        # chunk 2: i in [156,311) -- reads old mt[i+1], new mt[i-156]
        j = np.arange(_M, _N - 1)
        x2 = (mt[j] & _UM) | (mt[j + 1] & _LM)
        xa2 = (x2 >> one) ^ np.where((x2 & one) != 0, _A, np.uint64(0))
        new2 = new1[j - _M] ^ xa2
        # chunk 3: i = 311 -- reads new mt[0], new mt[155]
        x3 = (mt[_N - 1] & _UM) | (new1[0] & _LM)
        xa3 = (x3 >> one) ^ (_A if (int(x3) & 1) else np.uint64(0))
        new3 = new1[_N - 1 - _M] ^ xa3
        mt[0:_M] = new1
        mt[_M:_N - 1] = new2
        mt[_N - 1] = new3
        # tempering of the whole block
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self._buf = y
        self.idx = 0

    def next_u64_array(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        pos = 0
        while pos < n:
            if self.idx >= _N:
                self._twist()
            take = min(n - pos, _N - self.idx)
            out[pos:pos + take] = self._buf[self.idx:self.idx + take]
            self.idx += take
            pos += take
        return out

    def next_u64(self) -> int:
        return int(self.next_u64_array(1)[0])


class Substream:
    """rng.hpp:51-85."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)
        self.spare = 0.0
        self.have_spare = False

    def uniform01_array(self, n: int) -> np.ndarray:
        """rng.hpp:56 -- (x >> 11) * 2^-53, n draws in order."""
        u = self.eng.next_u64_array(n) >> np.uint64(11)
        return u.astype(np.float64) * (2.0 ** -53)

    def uniform01(self) -> float:
        return float(self.uniform01_array(1)[0])

    def normal(self, mu: float, sigma: float) -> float:
        """rng.hpp:59-72 Box-Muller with cached spare."""
        if self.have_spare:
            self.have_spare = False
            return mu + sigma * self.spare
        u1 = 0.0
        while u1 <= 0.0:
            u1 = self.uniform01()
        u2 = self.uniform01()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 2.0 * 3.14159265358979323846 * u2
        self.spare = r * math.sin(theta)
        self.have_spare = True
        return mu + sigma * r * math.cos(theta)

    def normal_array(self, n: int, mu: float, sigma: float) -> np.ndarray:
        """n sequential `normal` draws, vectorised.  Same draw order and
        operation order as normal(); numpy's vector sin/cos/log may differ
        from glibc in the last ulp, so use normal() where bit-equality with a
        C++ run matters (parity tests pass the generated data to both sides,
        so they never depend on this)."""
        out = np.empty(n, dtype=np.float64)
        pos = 0
        if self.have_spare and n > 0:
            out[0] = self.normal(mu, sigma)
            pos = 1
        pairs = (n - pos + 1) // 2
        if pairs > 0:
            u = self.uniform01_array(2 * pairs)
            u1, u2 = u[0::2], u[1::2]
            if np.any(u1 <= 0.0):  # astronomically rare: redo sequentially
                self.eng = None
                raise RuntimeError("u1 == 0 draw; use scalar normal()")
            r = np.sqrt(-2.0 * np.log(u1))
            theta = 2.0 * 3.14159265358979323846 * u2
            c = mu + (sigma * r) * np.cos(theta)  # C++ evaluates (sigma*r)*cos
            s = r * np.sin(theta)
            vals = np.empty(2 * pairs)
            vals[0::2] = c
            vals[1::2] = mu + sigma * s
            need = n - pos
            out[pos:] = vals[:need]
            if need < 2 * pairs:  # odd count: last spare stays cached
                self.spare = float(s[-1])
                self.have_spare = True
        return out

    def fill_uniform(self, rows: int, cols: int) -> np.ndarray:
        """rng.hpp:75-79 -- column by column (column-major order)."""
        return self.uniform01_array(rows * cols).reshape((rows, cols), order="F")
