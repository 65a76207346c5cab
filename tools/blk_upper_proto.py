#!/usr/bin/env python
"""Prototype (numpy, fp64) of the round-2 cfg4 kernel plan: the blocked
Cholesky + proposed inversion of SURVEY App. A.2 run on UPPER-TRIANGLE-ONLY storage, with
I3 replaced by G = C R_KT^H and V = -G R_KK^-H so that C can overwrite R_KT in place.

Storage rule checked here: every read and write touches W[i][j] with i <= j only (the lower
half of X_TT is read as the conjugate of the upper), so two matrices fit one square (one per
triangle).  Run: python tools/blk_upper_proto.py  (prints the max relative error vs numpy)."""
import numpy as np


class Upper:
    """n x n storage that only allows (i, j) with i <= j (asserts otherwise)."""

    def __init__(self, A):
        self.n = A.shape[0]
        self.w = np.triu(A).astype(complex)

    def get(self, i, j):
        assert i <= j, (i, j)
        return self.w[i, j]

    def set(self, i, j, v):
        assert i <= j, (i, j)
        self.w[i, j] = v

    def xt(self, m, j):                     # x~_mj of a Hermitian matrix stored upper
        return self.get(m, j) if m <= j else np.conj(self.get(j, m))


def factor(W, NB):
    """Crout panels (F1 / F2a / F2b): rows K of R from all previous rows, upper only."""
    n = W.n
    for k0 in range(0, n, NB):
        K = range(k0, k0 + NB)
        # F1: P_ij = a_ij - sum_{k<k0} conj(r_ki) r_kj, i in K, j >= i  (R rows k < k0, by rows)
        for i in K:
            for j in range(i, n):
                W.set(i, j, W.get(i, j) - sum(np.conj(W.get(k, i)) * W.get(k, j) for k in range(k0)))
        # F2a + F2b: right-looking within the panel rows
        for i in K:
            t = W.get(i, i).real
            assert t > 0
            r = np.sqrt(t)
            W.set(i, i, r)
            for j in range(i + 1, n):
                W.set(i, j, W.get(i, j) / r)
            for m in range(i + 1, k0 + NB):      # update the remaining panel rows
                for j in range(m, n):
                    W.set(m, j, W.get(m, j) - np.conj(W.get(i, m)) * W.get(i, j))


def invert(W, NB):
    """Blocked proposed inversion, panels from the bottom; I3 via G = C R_KT^H."""
    n = W.n
    for k0 in range(n - NB, -1, -NB):
        t0 = k0 + NB
        K, T = range(k0, t0), range(t0, n)
        # I1: C = R_KT X_TT (R_KT and X_TT both read from the upper storage)
        C = {(k, j): sum(W.get(k, m) * W.xt(m, j) for m in T) for k in K for j in T}
        # G = C R_KT^H (8 x 8 Hermitian), while R_KT is still in place
        G = np.array([[sum(C[(k, j)] * np.conj(W.get(kp, j)) for j in T) for kp in K] for k in K])
        # R_KK (upper, in place) and its reciprocals, kept before X overwrites the block
        RKK = np.array([[W.get(a, b) if a <= b else 0 for b in K] for a in K])
        # I2: rows K bottom-up, X_KT = -R_KK^-1 C, written over R_KT (C and R_KT consumed)
        for kk in reversed(range(NB)):
            k = k0 + kk
            for j in T:
                s = C[(k, j)] + sum(RKK[kk, mm] * W.get(k0 + mm, j) for mm in range(kk + 1, NB))
                W.set(k, j, -s / RKK[kk, kk])
        # V = -G R_KK^-H  (V_kj, k <= j used by I4)
        V = -G @ np.linalg.inv(RKK).conj().T if len(T) else np.zeros((NB, NB), complex)
        # I4: the diagonal block by the unblocked recursion with V added
        for kk in reversed(range(NB)):
            k = k0 + kk
            rk = RKK[kk]
            for jj in range(kk + 1, NB):
                s = V[kk, jj] + sum(rk[mm] * W.xt(k0 + mm, k0 + jj) for mm in range(kk + 1, NB))
                W.set(k, k0 + jj, -s / rk[kk])
            p = V[kk, kk].real + sum((rk[mm] * np.conj(W.get(k, k0 + mm))).real for mm in range(kk + 1, NB))
            ik = 1.0 / rk[kk].real
            W.set(k, k, ik * (ik - p))


def main():
    rng = np.random.default_rng(0)
    worst = 0.0
    for n, NB in ((8, 4), (16, 4), (16, 8), (32, 8), (64, 8)):
        G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        Q, _ = np.linalg.qr(G)
        lam = 10 ** (3 * rng.random(n))
        A = (Q * lam) @ Q.conj().T
        A = (A + A.conj().T) / 2
        W = Upper(A)
        factor(W, NB)
        invert(W, NB)
        X = np.triu(W.w) + np.triu(W.w, 1).conj().T
        Xe = np.linalg.inv(A)
        err = np.abs(X - Xe).max() / np.abs(Xe).max()
        worst = max(worst, err)
        print("n=%d NB=%d max rel err %.2e (cond %.1e)" % (n, NB, err, lam.max() / lam.min()))
    assert worst < 1e-10


if __name__ == "__main__":
    main()
