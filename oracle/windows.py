"""Canonical dual and canonical tight windows by the plain definition (test infrastructure).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Shares no code with the CUDA path.

The frame operator of the Gabor system G(g, Lambda) is S = sum_{lambda} <., pi(lambda) g>
pi(lambda) g (Eq. frameop, Sec. 2.1); the canonical dual window is S^{-1} g
and the canonical tight window S^{-1/2} g.  Lambda is the lattice of
Eq. (DGT): points (a n, b (m + w(n))) in the frequency units of PAPER.md:237 (m counted from
the lowest non-negative frequency), i.e. pi(lambda) g (l) = g((l - a n) mod L)
exp(2 pi i l (m + w(n)) / M), w(n) = (n lambda1 mod lambda2) / lambda2.  S is built densely
(L x L, numpy) from these atoms, the phases reduced exactly in integers; a library solve /
Hermitian eigendecomposition is the last step.  For small L only (L^2 M N / a work).
"""
from __future__ import annotations

import numpy as np


def synthesis_matrix(g, a: int, M: int, lam1: int, lam2: int) -> np.ndarray:
    """L x (M N) matrix whose column m N + n is the atom of coefficient c(m, n)."""
    g = np.asarray(g, dtype=np.complex128)
    L = g.shape[0]
    if L % a or L % M or (L // M) % lam2 or (L // a) % lam2 or not 0 <= lam1 < lam2:
        raise ValueError("infeasible lattice")
    N = L // a
    K = lam2 * M
    l = np.arange(L, dtype=np.int64)
    G = np.empty((L, M * N), dtype=np.complex128)
    for n in range(N):
        wp = (n * lam1) % lam2
        gs = g[(l - a * n) % L]
        for m in range(M):
            k = (l * (m * lam2 + wp)) % K          # exact: l (m + w(n)) / M = k / (lambda2 M) mod 1
            G[:, m * N + n] = gs * np.exp(2j * np.pi * k / K)
    return G


def frame_operator(g, a, M, lam1, lam2) -> np.ndarray:
    G = synthesis_matrix(g, a, M, lam1, lam2)
    return G @ G.conj().T


def canonical_dual(g, a, M, lam1, lam2) -> np.ndarray:
    """S^{-1} g."""
    return np.linalg.solve(frame_operator(g, a, M, lam1, lam2), np.asarray(g, dtype=np.complex128))


def canonical_tight(g, a, M, lam1, lam2) -> np.ndarray:
    """S^{-1/2} g."""
    ev, V = np.linalg.eigh(frame_operator(g, a, M, lam1, lam2))
    return (V * (1.0 / np.sqrt(ev))) @ (V.conj().T @ np.asarray(g, dtype=np.complex128))
