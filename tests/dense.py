"""Dense linear-algebra helpers for the oracle pins (tests only, tiny L).

Everything here is built from the operator definitions of the paper, NOT from
Eq. (DGT):  T_x f(l) = f(l - x), M_w f(l) = exp(2 pi i l w / L) f(l)
(Sec. 2.1), the lattice normal form [[a,0],[s,b]] with atoms
g_{n,k} = M_{sn+bk} T_{an} g (Prop. lattNF), the frame operator
S = sum <f, pi(lam) g> pi(lam) g (Eq. frameop) and the inversion
formula with the canonical dual S^{-1} g.  Phases here are
computed in floating point from the L-periodic definitions (independent of the
oracle's exact integer reduction).  The dense frame operator, canonical dual and tight
windows live in one place, oracle/windows.py (pinned in test_oracle_pins.py).
"""
from __future__ import annotations

import numpy as np


def lattice_points(L: int, a: int, M: int, lam1: int, lam2: int):
    """Yield (n, m, x, omega) for every lattice point, with m the Eq. (DGT) index.

    Points are (x, omega) = (a n, (s n + b k) mod L), s = b lam1/lam2.
    Following the indexing fixed at PAPER.md:237 ("counting the sampling points in
    frequency from the lowest nonnegative frequency upwards"), the frequency index
    of a point in column n is m = (omega - (s n mod b)) / b.
    """
    b = L // M
    N = L // a
    s = b * lam1 // lam2
    assert b * lam1 % lam2 == 0
    for n in range(N):
        base = (s * n) % b
        for k in range(M):
            om = (s * n + b * k) % L
            m = (om - base) // b
            assert (om - base) % b == 0
            yield n, m, a * n, om


def atom(g: np.ndarray, x: int, om: int) -> np.ndarray:
    """M_om T_x g."""
    L = len(g)
    l = np.arange(L)
    return np.exp(2j * np.pi * l * om / L) * g[(l - x) % L]


def synthesis_matrix(g: np.ndarray, a: int, M: int, lam1: int, lam2: int) -> np.ndarray:
    """L x (M*N) matrix whose column m*N + n is the atom of coefficient c(m, n)."""
    L = len(g)
    N = L // a
    G = np.zeros((L, M * N), dtype=np.complex128)
    for n, m, x, om in lattice_points(L, a, M, lam1, lam2):
        G[:, m * N + n] = atom(g.astype(np.complex128), x, om)
    return G


def dense_dgt(f, g, a, M, lam1, lam2) -> np.ndarray:
    """c = G^H f, reshaped to (M, N)."""
    L = len(g)
    G = synthesis_matrix(g, a, M, lam1, lam2)
    return (G.conj().T @ np.asarray(f, dtype=np.complex128)).reshape(M, L // a)


def synthesize(c: np.ndarray, gamma, a, M, lam1, lam2) -> np.ndarray:
    """f = sum_{m,n} c(m,n) M_{b(m+w(n))} T_{an} gamma."""
    G = synthesis_matrix(gamma, a, M, lam1, lam2)
    return G @ c.reshape(-1)
