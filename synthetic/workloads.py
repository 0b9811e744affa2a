"""Seeded synthetic workloads for the nonseparable-lattice DGT (arXiv:1307.4569).

This module is shared by the oracle side (tests, ``bench.py``'s cpu_baseline leg)
and the product side (tests, ``bench.py``).  It holds NO arithmetic of the method:
only the configuration table of ``BASELINE.json`` and the seeded generators for
the signal ``f`` and the window ``g``.  The recipe is DESIGN.md §3 (inputs) and
SURVEY.md §8(d):

* one independent PCG64 stream per signal, ``default_rng([seed_k, w])``, so any
  rank (or the oracle) can regenerate signal ``w`` alone;
* ``seed_k = 13074569 + k`` for config k (1-based);
* arrays are generated in fp64 and cast ONCE to the config dtype; the GPU path and
  the oracle consume the same bytes (the oracle upcasts them back to fp64);
* CN(0,1) = (z1 + i z2)/sqrt(2) with z1, z2 ~ N(0,1) (z1 drawn first, as one
  (2, L) block).

The window is the periodized Gaussian ``pgauss`` (reading Z14 of DESIGN.md): the
BASELINE.json formula is garbled, only "tfr = a*M/L" is explicit; we use
g(l) ∝ sum_{k=-3}^{3} exp(-pi (l + kL)^2 / (tfr L)), normalised to ||g||_2 = 1,
which is real and even.  The paper itself (Fig. 2) names no
test signal or window, so these stand in for "signals shaped like the paper's
workloads" (L a multiple of lcm(a,M), quincunx and lambda=1/3 lattices as in
PAPER.md:244-262, Fig. 1).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

SEED_BASE = 13074569


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (1-based index ``k``)."""

    k: int
    name: str
    L: int
    a: int
    M: int
    lam1: int
    lam2: int
    W: int
    dtype: str          # "c64" | "c128"  (working/output precision)
    real_input: bool    # f is real (promoted to complex on load)
    tfr_scale: float    # tfr = tfr_scale * a * M / L
    signal: str         # "real_normal" | "cn" | "chirps"

    @property
    def N(self) -> int:
        return self.L // self.a

    @property
    def b(self) -> int:
        return self.L // self.M

    @property
    def seed(self) -> int:
        return SEED_BASE + self.k

    @property
    def tfr(self) -> float:
        return self.tfr_scale * self.a * self.M / self.L

    @property
    def coefs_per_signal(self) -> int:
        return self.M * self.N


CONFIGS = [
    Workload(1, "cfg1_L240_quincunx_f64real", 240, 8, 12, 1, 2, 1, "c128", True, 1.0, "real_normal"),
    Workload(2, "cfg2_L144000_quincunx_c128", 144000, 50, 200, 1, 2, 1, "c128", False, 1.0, "cn"),
    Workload(3, "cfg3_L65536_quincunx_c64_W256", 65536, 64, 256, 1, 2, 256, "c64", False, 1.0, "chirps"),
    Workload(4, "cfg4_L737280_third_c128_W16", 737280, 60, 240, 1, 3, 16, "c128", False, 2.0, "cn"),
    Workload(5, "cfg5_L262144_quincunx_c64_W1024", 262144, 128, 512, 1, 2, 1024, "c64", False, 1.0, "cn"),
]


def config(k: int) -> Workload:
    return CONFIGS[k - 1]


def np_dtype(dtype: str, real: bool = False):
    if dtype == "c64":
        return np.float32 if real else np.complex64
    if dtype == "c128":
        return np.float64 if real else np.complex128
    raise ValueError(dtype)


def pgauss(L: int, tfr: float) -> np.ndarray:
    """Periodized Gaussian window in fp64, unit l2 norm, real and even (Z14)."""
    l = np.arange(L, dtype=np.float64)
    g = np.zeros(L, dtype=np.float64)
    for k in range(-3, 4):
        g += np.exp(-math.pi * (l + k * L) ** 2 / (tfr * L))
    g /= np.linalg.norm(g)
    return g


def window(wl: Workload) -> np.ndarray:
    """The config's window, cast once to the config dtype (always complex)."""
    return pgauss(wl.L, wl.tfr).astype(np_dtype(wl.dtype))


def _signal_fp64(kind: str, L: int, seed: int, w: int) -> np.ndarray:
    rng = np.random.default_rng([seed, w])
    if kind == "real_normal":
        return rng.standard_normal(L)
    if kind == "cn":
        z = rng.standard_normal((2, L))
        return (z[0] + 1j * z[1]) / math.sqrt(2.0)
    if kind == "chirps":
        phi = rng.random(8)
        nu0 = rng.random(8)
        nu1 = rng.random(8)
        z = rng.standard_normal((2, L))
        l = np.arange(L, dtype=np.float64)
        f = 0.1 * (z[0] + 1j * z[1]) / math.sqrt(2.0)
        for k in range(8):
            ph = phi[k] + nu0[k] * l + (nu1[k] - nu0[k]) * l * l / (2.0 * L)
            ph = ph - np.floor(ph)
            f = f + np.exp(2j * math.pi * ph)
        return f
    raise ValueError(kind)


def signal(wl: Workload, w: int) -> np.ndarray:
    """Signal ``w`` of config ``wl`` cast to the config dtype (real for real_input)."""
    x = _signal_fp64(wl.signal, wl.L, wl.seed, w)
    return x.astype(np_dtype(wl.dtype, wl.real_input))


def batch(wl: Workload, w0: int, w1: int, out: np.ndarray | None = None,
          threads: int = 8) -> np.ndarray:
    """Signals [w0, w1) as a contiguous (w1-w0, L) array (optionally into ``out``)."""
    n = w1 - w0
    if out is None:
        out = np.empty((n, wl.L), dtype=np_dtype(wl.dtype, wl.real_input))

    def fill(i):
        out[i] = signal(wl, w0 + i)

    if n > 1 and threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(fill, range(n)))
    else:
        for i in range(n):
            fill(i)
    return out


def random_pair(L: int, seed: int, dtype: str = "c128", real_f: bool = False):
    """Generic seeded (f, g) for parity sweeps on arbitrary lattices."""
    rng = np.random.default_rng([SEED_BASE, seed, L])
    if real_f:
        f = rng.standard_normal(L)
    else:
        z = rng.standard_normal((2, L))
        f = (z[0] + 1j * z[1]) / math.sqrt(2.0)
    z = rng.standard_normal((2, L))
    g = (z[0] + 1j * z[1]) / math.sqrt(2.0)
    g /= np.linalg.norm(g)
    return f.astype(np_dtype(dtype, real_f)), g.astype(np_dtype(dtype))
