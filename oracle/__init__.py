"""CPU oracle for the forward DGT on a nonseparable lattice (arXiv:1307.4569).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this package.
It shares no code with the CUDA path (``paper_1307_4569_b200``) and never imports it.

The oracle is the plain definition Eq. (DGT), PAPER.md:238-242 (Sec. 2.1), under
the DESIGN.md readings Z1 (0-based window shift) and Z2 (frequency index from the
lowest non-negative frequency).  See ``dgt_oracle.c`` for the two evaluations
(O1 literal sum, O2 regrouped sum).  Pins: ``tests/test_oracle_pins.py``.

``idgt`` is the synthesis operator (the inverse DGT with a dual window, the inversion
formula of PAPER.md:171-175), the adjoint of Eq. (DGT).

``windows.canonical_dual`` / ``windows.canonical_tight`` (numpy, dense frame operator of
Eq. frameop) give the dual and tight windows for small L.

Parity pinned for: ``dgt`` and ``idgt`` (both variants each), ``windows`` (S gamma = g through
dgt/idgt, perfect reconstruction, tight energy identity; tests/test_oracle_pins.py).  Nothing here is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import windows  # noqa: F401  (dense dual / tight windows)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dgt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (IEEE semantics: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        for name in ("oracle_dgt_literal", "oracle_dgt_regrouped"):
            fn = getattr(lib, name)
            fn.argtypes = [P, P, I, I, I, I, I, I, P, I, P, ctypes.c_int]
            fn.restype = ctypes.c_int
        for name in ("oracle_idgt_literal", "oracle_idgt_regrouped"):
            fn = getattr(lib, name)
            fn.argtypes = [P, P, I, I, I, I, I, I, P, ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def threads() -> int:
    return int(_load().oracle_threads())


def dgt(f, g, a: int, M: int, lam1: int, lam2: int, cols=None, variant: str = "auto",
        nthreads: int = 0) -> np.ndarray:
    """c[w, m, i] = c_w(m, cols[i]) of Eq. (DGT), computed in fp64.

    ``f``: (L,) or (W, L) real or complex; ``g``: (L,) real or complex.  Inputs are
    upcast exactly to complex128.  ``cols``: column indices n (None = all N).
    ``variant``: "literal" (O1), "regrouped" (O2) or "auto" (O2 unless L*M is tiny).
    Returns complex128 of shape (W, M, ncols) (or (M, ncols) for 1-D f).
    """
    lib = _load()
    f = np.asarray(f)
    squeeze = f.ndim == 1
    f2 = np.ascontiguousarray(np.atleast_2d(f), dtype=np.complex128)
    g2 = np.ascontiguousarray(np.asarray(g), dtype=np.complex128)
    W, L = f2.shape
    if g2.shape != (L,):
        raise ValueError("g must have length L")
    N = L // a if a > 0 else 0
    if cols is None:
        cols_arr = None
        ncols = N
    else:
        cols_arr = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
        ncols = int(cols_arr.size)
    c = np.zeros((W, M, ncols), dtype=np.complex128)
    if variant == "auto":
        variant = "literal" if L * M <= 4096 else "regrouped"
    fn = lib.oracle_dgt_literal if variant == "literal" else lib.oracle_dgt_regrouped
    rc = fn(f2.ctypes.data, g2.ctypes.data, L, a, M, lam1, lam2, W,
            None if cols_arr is None else cols_arr.ctypes.data, ncols, c.ctypes.data, int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (status {rc}): L={L} a={a} M={M} "
                         f"lambda={lam1}/{lam2}")
    return c[0] if squeeze else c


def idgt(c, gamma, a: int, M: int, lam1: int, lam2: int, variant: str = "auto",
         nthreads: int = 0) -> np.ndarray:
    """f[w, l] = sum_{m,n} c_w(m,n) gamma((l - a n) mod L) exp(2 pi i l (m + w(n)) / M), fp64.

    ``c``: (M, N) or (W, M, N); ``gamma``: (L,) synthesis window (the canonical dual of the
    analysis window inverts Eq. (DGT)).  ``variant``: "literal" (S1), "regrouped" (S2) or
    "auto".  Returns complex128 (L,) or (W, L).
    """
    lib = _load()
    c = np.asarray(c)
    squeeze = c.ndim == 2
    c3 = np.ascontiguousarray(c[None] if squeeze else c, dtype=np.complex128)
    g2 = np.ascontiguousarray(np.asarray(gamma), dtype=np.complex128)
    L = g2.shape[0]
    W, Mc, N = c3.shape
    if Mc != M or a <= 0 or N * a != L:
        raise ValueError("c must have shape (W, M, L/a)")
    f = np.zeros((W, L), dtype=np.complex128)
    if variant == "auto":
        variant = "literal" if L * M * N <= 1 << 22 else "regrouped"
    fn = lib.oracle_idgt_literal if variant == "literal" else lib.oracle_idgt_regrouped
    rc = fn(c3.ctypes.data, g2.ctypes.data, L, a, M, lam1, lam2, W, f.ctypes.data, int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (status {rc}): L={L} a={a} M={M} "
                         f"lambda={lam1}/{lam2}")
    return f[0] if squeeze else f
