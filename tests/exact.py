"""Exact Gaussian-rational arithmetic for test pins (no floating point, no oracle code).

Complex rationals are (Fraction re, Fraction im) pairs.  Used for brute-force Gauss-Jordan
inverses (X = A^-1 is defined by A X = I) and for closed-form exact families.
"""
from fractions import Fraction
from math import comb


def cadd(a, b):
    return (a[0] + b[0], a[1] + b[1])


def csub(a, b):
    return (a[0] - b[0], a[1] - b[1])


def cmul(a, b):
    return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])


def cconj(a):
    return (a[0], -a[1])


def cdiv(a, b):
    den = b[0] * b[0] + b[1] * b[1]
    num = cmul(a, cconj(b))
    return (num[0] / den, num[1] / den)


def to_exact(z):
    z = complex(z)
    return (Fraction(z.real), Fraction(z.imag))


def gauss_jordan_inverse(A):
    """Exact inverse of a square matrix of complex numbers/ints (list of lists)."""
    n = len(A)
    M = [[to_exact(A[i][j]) for j in range(n)] + [(Fraction(int(i == j)), Fraction(0))
                                                  for j in range(n)] for i in range(n)]
    zero = (Fraction(0), Fraction(0))
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != zero)
        M[col], M[piv] = M[piv], M[col]
        p = M[col][col]
        M[col] = [cdiv(v, p) for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != zero:
                f = M[r][col]
                M[r] = [csub(v, cmul(f, w)) for v, w in zip(M[r], M[col])]
    return [[M[i][n + j] for j in range(n)] for i in range(n)]


def exact_to_complex(X):
    return [[complex(float(v[0]), float(v[1])) for v in row] for row in X]


def pascal(n):
    """Symmetric Pascal matrix P_ij = C(i+j, i) (0-based).  Its Cholesky factor is the upper
    binomial matrix R_ij = C(j, i) (unit diagonal, so d = 1 in LDL)."""
    return [[comb(i + j, i) for j in range(n)] for i in range(n)]


def pascal_inverse(n):
    """P^-1 = R^-1 R^-*, with (R^-1)_ij = (-1)^(i+j) C(j, i) for j >= i; exact integers."""
    Ri = [[((-1) ** (i + j)) * comb(j, i) if j >= i else 0 for j in range(n)] for i in range(n)]
    return [[sum(Ri[i][p] * Ri[j][p] for p in range(n)) for j in range(n)] for i in range(n)]


def bidiag_family(c):
    """R unit upper bidiagonal with superdiagonal c (Gaussian integers).  Returns
    (A = R*R, X = A^-1) as exact Gaussian-integer lists: (R^-1)_ij = prod_{k=i}^{j-1} (-c_k)."""
    n = len(c) + 1
    R = [[0j] * n for _ in range(n)]
    for i in range(n):
        R[i][i] = 1 + 0j
        if i + 1 < n:
            R[i][i + 1] = complex(c[i])
    A = [[sum(R[k][i].conjugate() * R[k][j] for k in range(n)) for j in range(n)]
         for i in range(n)]
    Ri = [[0j] * n for _ in range(n)]
    for i in range(n):
        v = 1 + 0j
        Ri[i][i] = v
        for j in range(i + 1, n):
            v = v * (-complex(c[j - 1]))
            Ri[i][j] = v
    X = [[sum(Ri[i][p] * Ri[j][p].conjugate() for p in range(n)) for j in range(n)]
         for i in range(n)]
    return A, X
