"""Pins of the fixed-point oracle (readings F1-F7), no GPU.

What fixes it from outside itself: SPEC.md's worked quantize / fxp_mul examples,
exact identities and exactly representable cases, exact integer arithmetic checked against
Python's big integers, the wide-format bridge to the fp64 oracle (at very wide
formats the fixed-point result converges to the double-precision one), monotonicity of the
error in the fraction bits and determinism."""
import math

import numpy as np
import pytest
import torch

from paper_1111_4144_b200 import workloads as wl

Q213 = (2, 13)


def test_spec_quantize_examples():
    # quantize(0.0) = 0; quantize(0.3, f=2) -> raw 1; quantize(5.0, m=1, f=2) -> raw 7
    assert wl.quantize(torch.tensor([0.0]), 2, 13).item() == 0
    assert wl.quantize(torch.tensor([0.3]), 2, 2).item() == 1
    assert wl.quantize(torch.tensor([5.0]), 1, 2).item() == 7
    assert wl.quantize(torch.tensor([-9.0]), 1, 2).item() == -8           # lower bound -2^m
    assert wl.quantize(torch.tensor([0.375, 0.125]), 2, 2).tolist() == [2, 0]   # ties to even


def test_spec_fxp_mul_examples(orc):
    # S:84-86 with f = 2 (raw = value * 4): 1 * z = z; 0.5 * 0.5 = 0.25; (0.75+0.5i)(0.75-0.5i) -> 0.75
    z, ns = orc.fxp_op("mul", 2, 2, (4, 0), (3, -2))
    assert z == (3, -2) and ns == 0
    z, _ = orc.fxp_op("mul", 2, 4, (8, 0), (8, 0))                  # f = 4: 0.5 * 0.5
    assert z == (4, 0)
    z, _ = orc.fxp_op("mul", 2, 2, (3, 2), (3, -2))                  # 13/16 -> 3/4 (raw 3)
    assert z == (3, 0)
    z, ns = orc.fxp_op("mul", 1, 2, (7, 0), (7, 0))                  # 1.75^2 saturates at 1.75
    assert z == (7, 0) and ns == 1


def test_fxp_ops_against_big_integers(orc):
    """F4-F6 on random raws: exact rational results rounded half-to-even (Python integers)."""
    rng = np.random.default_rng(0)
    m, f = 3, 20
    lo, hi = -(1 << (m + f)), (1 << (m + f)) - 1

    def rne_div(num, den):                                         # den > 0, exact
        q, r = divmod(num, den)
        return q + 1 if (2 * r > den or (2 * r == den and q % 2 == 1)) else q

    def clamp(v):
        return max(lo, min(hi, v))
    for _ in range(300):
        a = [int(v) for v in rng.integers(-(1 << 21), 1 << 21, 2)]
        b = [int(v) for v in rng.integers(-(1 << 21), 1 << 21, 2)]
        z, _ = orc.fxp_op("mul", m, f, a, b)
        re = a[0] * b[0] - a[1] * b[1]
        im = a[0] * b[1] + a[1] * b[0]
        assert z == (clamp(rne_div(re, 1 << f)), clamp(rne_div(im, 1 << f)))
        p = int(rng.integers(1, 1 << 22))
        z, _ = orc.fxp_op("div", m, f, a, (p, 0))
        assert z == (clamp(rne_div(a[0] << f, p)), clamp(rne_div(a[1] << f, p)))
        t = int(rng.integers(1, 1 << 23))
        z, _ = orc.fxp_op("sqrt", m, f, (t, 0))
        x = t << f
        r = math.isqrt(x)
        r = r + 1 if x - r * r > r else r
        assert z[0] == clamp(r)


def _raw(A, m, f):
    A = torch.as_tensor(A, dtype=torch.complex128)
    return torch.stack([wl.quantize(A.real, m, f), wl.quantize(A.imag, m, f)], -1).numpy()


@pytest.mark.parametrize("method", ["proposed", "eqsolve", "trimat"])
def test_identity_and_exact_families(orc, method):
    # identity and diag(2, 1/2, 1, 4 - ...) -> reciprocals exact where representable
    for n in (1, 2, 5, 16):
        X, info, ns = orc.fxp_inv_batched(_raw(np.eye(n)[None], *Q213), *Q213, method)
        assert info[0] == 0 and ns[0] == 0
        assert np.array_equal(X[0, ..., 0], np.eye(n) * (1 << 13)) and not X[0, ..., 1].any()
    # unit upper bidiagonal {+-1, +-i} family: A = R*R, X Gaussian integers with |x| <= n:
    # exact in Q5.13 (every intermediate is a small Gaussian integer)
    rng = np.random.default_rng(3)
    units = np.array([1, -1, 1j, -1j])
    n = 6
    As, Xs = [], []
    for _ in range(20):
        R = np.eye(n, dtype=complex)
        R[np.arange(n - 1), np.arange(1, n)] = units[rng.integers(0, 4, n - 1)]
        A = R.conj().T @ R
        As.append(A)
        Xs.append(np.linalg.inv(A))
    X, info, ns = orc.fxp_inv_batched(_raw(np.array(As), 5, 13), 5, 13, method)
    assert (info == 0).all() and (ns == 0).all()
    Xe = np.round(np.array(Xs).real) + 1j * np.round(np.array(Xs).imag)
    assert np.array_equal(X[..., 0] / 8192.0 + 1j * X[..., 1] / 8192.0, Xe)


def _study(orc, method, m, f, n=16, count=200):
    cfg = wl.Config(8, n, torch.complex128, count, "chol", "aos", "fxp", float(n), 0.1, task="fxp", qm=m, qf=f)
    A, raw = wl.generate_fxp(cfg, 0, count)
    X, info, ns = orc.fxp_inv_batched(raw.numpy(), m, f, method)
    Xr = np.linalg.inv(A.numpy())
    Xf = X[..., 0] / 2.0 ** f + 1j * X[..., 1] / 2.0 ** f
    ok = (info == 0) & (ns == 0)
    err = np.linalg.norm((Xf - Xr)[ok], axis=(1, 2)) / np.linalg.norm(Xr[ok], axis=(1, 2))
    return err, ok


@pytest.mark.parametrize("method", ["proposed", "eqsolve", "trimat"])
def test_wide_format_bridge_to_double(orc, method):
    """at a very wide format the fixed-point result is the double-precision one."""
    err, ok = _study(orc, method, 9, 31, n=8, count=50)
    assert ok.all() and err.max() <= 1e-6


@pytest.mark.parametrize("method", ["proposed", "eqsolve", "trimat"])
def test_error_decreases_with_fraction_bits(orc, method):
    """S:400 / S:474: mean relative error non-increasing over f in {8, 13, 23} (5% noise)."""
    means = []
    for f in (8, 13, 23):
        err, ok = _study(orc, method, 6, f, n=8, count=100)
        assert ok.mean() > 0.9
        means.append(err.mean())
    assert means[1] <= 1.05 * means[0] and means[2] <= 1.05 * means[1], means


def test_determinism_and_failures(orc):
    cfg = wl.CONFIGS[8]
    _, raw = wl.generate_fxp(cfg, 0, 30)
    r = raw.numpy().copy()
    r[3] = 0                                     # zero matrix: pivot 1 fails
    X1, i1, s1 = orc.fxp_inv_batched(r, *Q213, "proposed", nthreads=1)
    X2, i2, s2 = orc.fxp_inv_batched(r, *Q213, "proposed")
    assert np.array_equal(X1, X2) and np.array_equal(i1, i2) and np.array_equal(s1, s2)
    assert i1[3] == 1 and not X1[3].any()
