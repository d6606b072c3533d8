"""The five BASELINE.json configurations as seeded synthetic inputs.

Geometry, mesh, interface grid, loads and recovery points per
BASELINE.json `configs`; the generator recipe follows SURVEY.md §8(d):
uniform linspace grids, liner E = 71.7 GPa, per-block dT_b = -270 + 40 u_b
and dummy iff u_b < 0.2 with u_b = (mt19937_64(seed)() >> 11) * 2^-53 in
cell order (std::uniform_real_distribution is library-dependent, so it
is not used).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

DT_SEED = 2411       # config 3 per-block dT
DUMMY_SEED = 12690   # config 4 Bernoulli(0.2) dummy sites


class MT19937_64:
    """std::mt19937_64 (Matsumoto & Nishimura 64-bit Mersenne Twister,
    the parameters fixed by the C++ standard [rand.predef])."""
    _N, _M = 312, 156
    _MASK = (1 << 64) - 1
    _UPPER, _LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self._N
        mt[0] = seed & self._MASK
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & self._MASK
        self.mt, self.idx = mt, self._N

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        for i in range(N):
            y = (mt[i] & self._UPPER) | (mt[(i + 1) % N] & self._LOWER)
            v = mt[(i + M) % N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self._N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK


def uniform01(seed: int, count: int) -> np.ndarray:
    g = MT19937_64(seed)
    return np.array([(g() >> 11) * 2.0 ** -53 for _ in range(count)], np.float64)


@dataclass(frozen=True)
class TsvConfig:
    name: str
    rows: int
    cols: int
    d: float
    h: float
    t: float
    p: float
    m_xy: int           # cells per axis in x/y (uniform)
    m_z: int            # cells along z
    q: int              # interpolation nodes per axis (p + 1)
    points: int         # 8 = 2x2x2 Gauss, 1 = centroid
    dt_uniform: Optional[float] = -250.0
    dt_seed: Optional[int] = None
    dummy_fraction: float = 0.0
    dummy_seed: Optional[int] = None
    liner_e: float = 71.7e9

    @property
    def B(self):
        return self.rows * self.cols

    @property
    def n(self):
        q = self.q
        return 3 * (q ** 3 - (q - 2) ** 3)

    @property
    def n_fine(self):
        return 3 * (self.m_xy + 1) ** 2 * (self.m_z + 1)

    @property
    def elements(self):
        return self.m_xy * self.m_xy * self.m_z

    def delta_t(self) -> np.ndarray:
        if self.dt_seed is not None:
            return -270.0 + 40.0 * uniform01(self.dt_seed, self.B)
        return np.array([self.dt_uniform], np.float64)

    def kinds(self) -> Optional[np.ndarray]:
        if self.dummy_seed is None:
            return None
        return (uniform01(self.dummy_seed, self.B) < self.dummy_fraction).astype(np.uint8)

    def materials(self) -> np.ndarray:
        """[3,3] E, nu, alpha: Cu / SiO2 liner / Si (material.cpp:37-43, liner E overridden)."""
        return np.array([[110e9, 0.35, 17e-6], [self.liner_e, 0.16, 0.5e-6], [130e9, 0.28, 2.8e-6]])

    def lattice_dofs(self) -> int:
        q, B = self.q, self.B
        lat_x, lat_y = self.cols * (q - 1) + 1, self.rows * (q - 1) + 1
        return 3 * (lat_x * lat_y * q - B * (q - 2) ** 3)


_G0 = dict(d=5e-6, h=50e-6, t=0.5e-6, p=15e-6)
_G2 = dict(d=4e-6, h=40e-6, t=0.4e-6, p=10e-6)

CONFIGS = [
    TsvConfig("cfg0_3x3", 3, 3, m_xy=16, m_z=16, q=5, points=8, **_G0),
    TsvConfig("cfg1_10x10", 10, 10, m_xy=16, m_z=16, q=5, points=8, **_G0),
    TsvConfig("cfg2_32x32", 32, 32, m_xy=24, m_z=24, q=6, points=8, **_G2),
    TsvConfig("cfg3_100x100", 100, 100, m_xy=20, m_z=20, q=7, points=8, dt_uniform=None, dt_seed=DT_SEED, **_G0),
    TsvConfig("cfg4_200x200", 200, 200, m_xy=16, m_z=16, q=5, points=1, dummy_fraction=0.2,
              dummy_seed=DUMMY_SEED, **_G0),
]


def get(i_or_name) -> TsvConfig:
    if isinstance(i_or_name, int):
        return CONFIGS[i_or_name]
    for c in CONFIGS:
        if c.name == i_or_name or c.name.startswith(str(i_or_name)):
            return c
    raise KeyError(i_or_name)
