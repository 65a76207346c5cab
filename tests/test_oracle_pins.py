"""Pins for the fp64 oracle against things other than itself (CPU only).

Each pin is chosen so that a plausible mistake in the oracle (a dropped term, a missing
conjugate, a wrong sign or index, a transposed operand) fails at least one of them:
closed forms, exact-integer families, exact Gaussian-rational Gauss-Jordan, LAPACK, the
paper's structural theorem behind eq. (24), and the worked examples.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla

from tests import exact

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cplx(a):
    a = np.asarray(a, dtype=np.float64)
    return a[..., 0] + 1j * a[..., 1]


def rand_hpd(rng, n, delta=0.1):
    B = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    A = B @ B.conj().T / n + delta * np.eye(n)
    A = (A + A.conj().T) / 2
    return A


def invert(orc, A, method):
    if method == "ldl":
        R, d, info = orc.ldl_upper(A)
        assert info == 0
        return orc.proposed_inv_ldl(R, d)
    R, info = orc.chol_upper(A)
    assert info == 0
    if method == "chol":
        return orc.proposed_inv_chol(R)
    if method == "eqsolve":
        return orc.eqsolve_inv(R)
    return orc.trimat_inv(R)


ALL = ["chol", "ldl", "eqsolve", "trimat"]


# ------------------------------------------------------------------ worked examples (golden)
def test_worked_examples(orc):
    g = json.load(open(os.path.join(GOLD, "worked_examples.json")))
    for case in g["cholesky"]:
        R, info = orc.chol_upper(cplx(case["A"]))
        assert info == case["info"], case["cite"]
        if info == 0:
            np.testing.assert_allclose(R, cplx(case["R"]), rtol=0, atol=1e-15, err_msg=case["cite"])
    for case in g["ldl"]:
        R, d, info = orc.ldl_upper(cplx(case["A"]))
        assert info == case["info"]
        np.testing.assert_allclose(R, cplx(case["R"]), atol=1e-15)
        np.testing.assert_allclose(d, case["d"], atol=1e-15)
    for case in g["inverse"]:
        for m in ALL:
            X = invert(orc, cplx(case["A"]), m)
            np.testing.assert_allclose(X, cplx(case["X"]), rtol=2e-15, atol=1e-16, err_msg=case["cite"])


def test_gauss_jordan_golden(orc):
    """Exact Gaussian-rational inverses of integer HPD matrices (tests/golden/make_golden.py)."""
    g = json.load(open(os.path.join(GOLD, "gauss_jordan.json")))
    for case in g["cases"]:
        A = np.array(case["A_re"], float) + 1j * np.array(case["A_im"], float)
        Xe = (np.array([[float(Fraction(v)) for v in r] for r in case["X_re"]])
              + 1j * np.array([[float(Fraction(v)) for v in r] for r in case["X_im"]]))
        for m in ALL:
            X = invert(orc, A, m)
            assert np.abs(X - Xe).max() <= 1e-14 * np.abs(Xe).max(), (m, case["n"])


# --------------------------------------------------------------------------- closed forms
def test_2x2_closed_form(orc):
    """[[a,b],[conj b,c]]^-1 = [[c,-b],[-conj b,a]]/(ac-|b|^2); complex b catches a
    missing/misplaced conjugate anywhere in eqs. 3-4, 10-11 or the back-substitution."""
    rng = np.random.default_rng(1)
    for _ in range(50):
        a, c = rng.uniform(1, 3, 2)
        b = complex(*rng.uniform(-0.9, 0.9, 2))
        A = np.array([[a, b], [np.conj(b), c]])
        det = a * c - abs(b) ** 2
        Xe = np.array([[c, -b], [-np.conj(b), a]]) / det
        for m in ALL:
            np.testing.assert_allclose(invert(orc, A, m), Xe, rtol=1e-14, atol=1e-15)


def test_diagonal_and_identity(orc):
    for n in (1, 2, 5, 17):
        v = np.arange(1, n + 1, dtype=float) * 1.5
        for m in ALL:
            X = invert(orc, np.diag(v), m)
            np.testing.assert_allclose(X, np.diag(1 / v), rtol=1e-15, atol=0)
            assert np.array_equal(invert(orc, np.eye(n), m), np.eye(n))


@pytest.mark.parametrize("n", [1, 2, 3, 6, 12, 20, 24])
def test_pascal_exact(orc, n):
    """Pascal P_ij = C(i+j,i): R_ij = C(j,i), d = 1, X exact integers (fp64-exact to n=24)."""
    P = np.array(exact.pascal(n), dtype=float)
    Xe = np.array(exact.pascal_inverse(n), dtype=float)
    R, info = orc.chol_upper(P)
    assert info == 0
    Re = np.array([[float(__import__("math").comb(j, i)) if j >= i else 0 for j in range(n)]
                   for i in range(n)])
    assert np.array_equal(R, Re)
    R2, d, info = orc.ldl_upper(P)
    assert info == 0 and np.array_equal(R2, Re) and np.array_equal(d, np.ones(n))
    for m in ALL:
        assert np.array_equal(invert(orc, P, m), Xe), m


@pytest.mark.parametrize("n", [3, 8, 12])
def test_complex_pascal_similarity_exact(orc, n):
    """U = diag(i^k): A' = U P U^H has R' = U R U^H and X' = U X U^H exactly.  Real Pascal
    cannot see a missing conjugate; this complex version can."""
    P = np.array(exact.pascal(n), dtype=float)
    Xe = np.array(exact.pascal_inverse(n), dtype=float)
    u = np.array([1j ** k for k in range(n)])
    u = np.round(u.real) + 1j * np.round(u.imag)
    Ap = (u[:, None] * P) * np.conj(u)[None, :]
    Xp = (u[:, None] * Xe) * np.conj(u)[None, :]
    for m in ALL:
        assert np.array_equal(invert(orc, Ap, m), Xp), m


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_unit_bidiagonal_family_exact(orc, n):
    """R unit upper bidiagonal, superdiagonal in {+-1, +-i}: A = R*R and X are Gaussian
    integers, so every method must be bit-exact in fp64 (for all n <= 64)."""
    rng = np.random.default_rng(n)
    units = [1, -1, 1j, -1j]
    c = [units[k] for k in rng.integers(0, 4, n - 1)]
    A, X = exact.bidiag_family(c)
    A, X = np.array(A), np.array(X)
    for m in ALL:
        assert np.array_equal(invert(orc, A, m), X), m


@pytest.mark.parametrize("n", [4, 16, 64])
def test_kms_closed_form(orc, n):
    """KMS / AR(1): a_ij = rho^(j-i) (j >= i), complex |rho| < 1.  Closed forms: R row 0 =
    rho^j, row i>0 = sqrt(1-|rho|^2) rho^(j-i); LDL d = (1, 1-|rho|^2, ...), R_ij = rho^(j-i);
    X = tridiag(-conj(rho), [1, 1+|rho|^2, ..., 1], -rho) / (1-|rho|^2)."""
    rho = 0.55 * np.exp(0.7j)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    up = rho ** np.maximum(j - i, 0)
    A = np.where(j >= i, up, np.conj(rho ** np.maximum(i - j, 0)))
    s = np.sqrt(1 - abs(rho) ** 2)
    Re = np.where(j >= i, up, 0) * np.where(i == 0, 1.0, s)
    R, info = orc.chol_upper(A)
    assert info == 0
    np.testing.assert_allclose(R, Re, atol=1e-14)
    R2, d, _ = orc.ldl_upper(A)
    np.testing.assert_allclose(R2, np.where(j >= i, up, 0), atol=1e-14)
    np.testing.assert_allclose(d, [1.0] + [1 - abs(rho) ** 2] * (n - 1), atol=1e-14)
    Xe = np.zeros((n, n), complex)
    for k in range(n):
        Xe[k, k] = 1 + (abs(rho) ** 2 if 0 < k < n - 1 else 0)
        if k + 1 < n:
            Xe[k, k + 1] = -rho
            Xe[k + 1, k] = -np.conj(rho)
    Xe /= 1 - abs(rho) ** 2
    for m in ALL:
        np.testing.assert_allclose(invert(orc, A, m), Xe, atol=1e-13)


@pytest.mark.parametrize("n", [8, 64])
def test_spectral_closed_form(orc, n):
    """cfg4 construction A = Q diag(lam) Q^H  =>  X = Q diag(1/lam) Q^H."""
    rng = np.random.default_rng(7)
    G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    Q, _ = np.linalg.qr(G)
    lam = 10 ** rng.uniform(0, 3, n)
    A = (Q * lam) @ Q.conj().T
    A = (A + A.conj().T) / 2
    Xe = (Q / lam) @ Q.conj().T
    cond = lam.max() / lam.min()
    for m in ALL:
        X = invert(orc, A, m)
        assert np.abs(X - Xe).max() / np.abs(Xe).max() <= 1e-14 * cond


# ----------------------------------------------------------------- library special cases
@pytest.mark.parametrize("n", [1, 3, 8, 16, 33, 64])
def test_against_lapack(orc, n):
    """Cholesky factor vs LAPACK zpotrf (upper), inverse vs zpotri and numpy.linalg.inv."""
    rng = np.random.default_rng(100 + n)
    A = rand_hpd(rng, n)
    Rl, infl = sla.lapack.zpotrf(A, lower=0)
    assert infl == 0
    R, info = orc.chol_upper(A)
    np.testing.assert_allclose(R, np.triu(Rl), atol=1e-13)
    Xl, _ = sla.lapack.zpotri(Rl, lower=0)
    Xl = np.triu(Xl) + np.triu(Xl, 1).conj().T
    Xn = np.linalg.inv(A)
    for m in ALL:
        X = invert(orc, A, m)
        sc = np.abs(Xn).max()
        assert np.abs(X - Xl).max() <= 1e-12 * sc
        assert np.abs(X - Xn).max() <= 1e-12 * sc
        # residual ||AX - I||_F (SPEC acceptance 2)
        assert np.linalg.norm(A @ X - np.eye(n)) <= 1e-8


def test_cross_method_agreement(orc):
    rng = np.random.default_rng(3)
    for n in (5, 16, 32):
        A = rand_hpd(rng, n)
        R, _ = orc.chol_upper(A)
        Xs = [invert(orc, A, m) for m in ALL]
        Xs += [orc.eqsolve_inv(R, orc.FULL_EXPLOITATION), orc.trimat_inv(R, orc.FULL_EXPLOITATION)]
        for X in Xs[1:]:
            assert np.abs(X - Xs[0]).max() <= 1e-10 * np.abs(Xs[0]).max()


# --------------------------------------------------------- structure behind eqs. (22)-(24)
@pytest.mark.parametrize("n", [4, 16])
def test_shortcut_theorem(orc, n):
    """B = L^-1 (L = R*) is lower triangular with diagonal 1/l_ii: the S of eq. (24)
    is exactly the upper part of B.  Same for B~ = (R*D)^-1 and S~ = diag(1/d_i) (eq. 29)."""
    rng = np.random.default_rng(n)
    A = rand_hpd(rng, n)
    R, _ = orc.chol_upper(A)
    B = sla.solve_triangular(R.conj().T, np.eye(n), lower=True)
    assert np.abs(np.triu(B, 1)).max() == 0
    np.testing.assert_allclose(np.diag(B), 1 / np.diag(R), rtol=1e-15)
    R2, d, _ = orc.ldl_upper(A)
    Bt = sla.solve_triangular(R2.conj().T * d[None, :], np.eye(n), lower=True)
    assert np.abs(np.triu(Bt, 1)).max() == 0
    np.testing.assert_allclose(np.diag(Bt), 1 / d, rtol=1e-14)
    # R X = S: the proposed X satisfies the upper part of eq. (23) with B replaced by S
    X = orc.proposed_inv_chol(R)
    RX = R @ X
    np.testing.assert_allclose(np.triu(RX), np.diag(1 / np.diag(R).real), atol=1e-13)


def test_ldl_cholesky_relation(orc):
    """r_c,ii^2 = d_i and R_c = diag(sqrt d) R_l (eqs. 3-4 vs 10-11); reconstructions."""
    rng = np.random.default_rng(11)
    for n in (2, 9, 32):
        A = rand_hpd(rng, n)
        Rc, _ = orc.chol_upper(A)
        Rl, d, _ = orc.ldl_upper(A)
        np.testing.assert_allclose(np.diag(Rc).real ** 2, d, rtol=1e-13)
        np.testing.assert_allclose(Rc, np.sqrt(d)[:, None] * Rl, atol=1e-13)
        np.testing.assert_allclose(Rc.conj().T @ Rc, A, atol=1e-13)
        np.testing.assert_allclose(Rl.conj().T @ (d[:, None] * Rl), A, atol=1e-13)
        assert np.all(np.diag(Rl) == 1)


# ------------------------------------------------------------------------ info and mirror
def test_info_cases(orc):
    cases = [
        (np.array([[1, 2], [2, 1]], complex), 2),
        (np.diag([1.0, -1.0, 1.0]).astype(complex), 2),
        (np.zeros((3, 3), complex), 1),
        (np.eye(4, dtype=complex), 0),
    ]
    A = np.eye(4, dtype=complex) * 2
    A[2, 2] = np.nan
    cases.append((A, 3))
    A = np.eye(4, dtype=complex) * 2
    A[3, 1] = np.nan          # strictly lower: never read (reading R5)
    cases.append((A, 0))
    A = np.eye(4, dtype=complex) * 2
    A[1, 1] = 2 + 5j          # Im a_ii ignored
    cases.append((A, 0))
    A = np.eye(3, dtype=complex)
    A[2, 2] = -np.inf
    cases.append((A, 3))
    for A, want in cases:
        _, info = orc.chol_upper(A)
        assert info == want
        _, _, info = orc.ldl_upper(A)
        assert info == want
        X, infos = orc.inv_batched(A[None].copy(), "chol")
        assert infos[0] == want
        if want:
            assert np.isnan(X).all()


def test_mirror_invariants(orc):
    rng = np.random.default_rng(5)
    for n in (1, 7, 16):
        A = rand_hpd(rng, n)
        for m in ALL:
            X = invert(orc, A, m)
            assert np.array_equal(X, X.conj().T)
            assert np.all(np.diag(X).imag == 0)
    U = np.triu(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    M = orc.mirror(U)
    assert np.array_equal(M, M.conj().T) and np.array_equal(np.triu(M, 1), np.triu(U, 1))


# ------------------------------------------------------------------ linear solves (f1 row)
def test_solves(orc):
    rng = np.random.default_rng(9)
    for n in (1, 4, 16, 32):
        A = rand_hpd(rng, n)
        y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        xe = np.linalg.solve(A, y)
        R, _ = orc.chol_upper(A)
        np.testing.assert_allclose(orc.solve_chol(R, y), xe, atol=1e-12 * np.abs(xe).max())
        R2, d, _ = orc.ldl_upper(A)
        np.testing.assert_allclose(orc.solve_ldl(R2, d, y), xe, atol=1e-12 * np.abs(xe).max())
    # exact: Gaussian-integer family, y = A x with integer x recovers x bit-exactly
    c = [1, 1j, -1, -1j, 1j, 1, -1]
    A, _ = exact.bidiag_family(c)
    A = np.array(A)
    x = np.arange(1, 9) + 1j * np.arange(8, 0, -1)
    y = A @ x
    R, _ = orc.chol_upper(A)
    assert np.array_equal(orc.solve_chol(R, y), x)
    R2, d, _ = orc.ldl_upper(A)
    assert np.array_equal(orc.solve_ldl(R2, d, y), x)
    # SPEC.md:246 worked example: R = [[1,.5],[0,1]], d = (2,1.5), y = (2,2.5) -> b = (1,1)
    # so x = R^-1 b = (0.5, 1)
    x = orc.solve_ldl(np.array([[1, .5], [0, 1]]), [2, 1.5], np.array([2, 2.5]))
    np.testing.assert_allclose(x, [0.5, 1.0], atol=1e-15)


def test_nonhermitian(orc):
    """D^-1 = D* (DD*)^-1; SPEC.md:343-344 worked examples."""
    Di, info = orc.nonhermitian_inv(np.array([[0, 1], [1, 0]], complex))
    assert info == 0 and np.array_equal(Di, np.array([[0, 1], [1, 0]]))
    Di, _ = orc.nonhermitian_inv(np.array([[1, 1], [0, 1]], complex))
    np.testing.assert_allclose(Di, [[1, -1], [0, 1]], atol=1e-14)
    rng = np.random.default_rng(4)
    for n in (3, 8, 16):
        D = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 3 * np.eye(n)
        Di, info = orc.nonhermitian_inv(D)
        assert info == 0
        Xe = np.linalg.inv(D)
        assert np.abs(Di - Xe).max() <= 1e-10 * np.abs(Xe).max() * np.linalg.cond(D) ** 2 * 1e-2


def test_nonhermitian_batched(orc):
    """The batched driver equals per-matrix calls; on exactly invertible Gaussian-integer D
    (unit upper bidiagonal {+-1, +-i} times a signed permutation) D^-1 is checked against the
    exact inverse, and against numpy.linalg.inv on random D."""
    rng = np.random.default_rng(11)
    Ds = []
    for _ in range(20):
        n = 6
        U = np.eye(n, dtype=complex)
        U[np.arange(n - 1), np.arange(1, n)] = np.array([1, -1, 1j, -1j])[rng.integers(0, 4, n - 1)]
        P = np.eye(n)[rng.permutation(n)] * rng.choice([-1, 1], n)
        Ds.append(P @ U)
    Ds = np.array(Ds)
    Dinv, info = orc.nonherm_batched(Ds)
    assert (info == 0).all()
    for b in range(len(Ds)):
        np.testing.assert_allclose(Dinv[b] @ Ds[b], np.eye(6), atol=1e-12)
        one, i1 = orc.nonhermitian_inv(Ds[b])
        assert np.array_equal(one, Dinv[b]) and i1 == info[b]
    D = rng.standard_normal((7, 5, 5)) + 1j * rng.standard_normal((7, 5, 5)) + 2 * np.eye(5)
    Dinv, info = orc.nonherm_batched(D)
    np.testing.assert_allclose(Dinv, np.linalg.inv(D), rtol=0, atol=1e-11)
    Dz = np.zeros((1, 3, 3), complex)
    Dinv, info = orc.nonherm_batched(Dz)
    assert info[0] == 1 and np.isnan(Dinv).all()


# ---------------------------------------------------------------------- batched + strides
def test_batched_layouts(orc):
    """The strided batched driver equals the single-matrix routines, for AoS and SoA
    ("interleaved") layouts, and never reads the strict lower triangle."""
    rng = np.random.default_rng(12)
    n, batch = 5, 7
    As = np.stack([rand_hpd(rng, n) for _ in range(batch)])
    ref = np.stack([invert(orc, a, "chol") for a in As])
    # AoS with lower triangle poisoned
    aos = As.copy()
    il = np.tril_indices(n, -1)
    aos[:, il[0], il[1]] = np.nan
    X, info = orc.inv_batched(aos, "chol")
    assert (info == 0).all() and np.array_equal(X, ref)
    # SoA: planes of length ld >= batch; element (i,j) of b at base[b + (i*n+j)*ld]
    ld = 9
    soa = np.full((n * n, ld), np.nan + 0j)
    soa[:, :batch] = As.reshape(batch, n * n).T
    view = np.lib.stride_tricks.as_strided(soa, shape=(batch, n, n),
                                           strides=(16, n * ld * 16, ld * 16))
    X2, info2 = orc.inv_batched(view, "chol")
    assert np.array_equal(X2, ref)
    for m in ("ldl", "eqsolve", "trimat"):
        Xm, _ = orc.inv_batched(aos, m)
        assert np.abs(Xm - ref).max() <= 1e-12 * np.abs(ref).max()
    y = rng.standard_normal((batch, n)) + 0j
    x, info = orc.solve_batched(aos, y, "chol")
    np.testing.assert_allclose(np.einsum("bij,bj->bi", As, x), y, atol=1e-12)
