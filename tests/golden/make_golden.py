"""Writes tests/golden/gauss_jordan.json: exact inverses of small integer Hermitian PD
matrices by brute-force Gaussian-rational Gauss-Jordan (tests/exact.py).

Calls neither oracle/ nor the CUDA path: the expected values come from the definition
A X = I (eq. 15 / eq. 20) in exact arithmetic.  Re-run:
    python tests/golden/make_golden.py
"""
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from exact import gauss_jordan_inverse  # noqa: E402


def hpd_integer(n, rng):
    # A = G G* + n I with small Gaussian-integer G: Hermitian, integer, PD.
    G = [[complex(rng.randint(-2, 2), rng.randint(-2, 2)) for _ in range(n)] for _ in range(n)]
    A = [[sum(G[i][p] * G[j][p].conjugate() for p in range(n)) + (n if i == j else 0)
          for j in range(n)] for i in range(n)]
    return A


def main():
    rng = random.Random(20111144)
    cases = []
    for n in (1, 2, 3, 4):
        for t in range(3):
            A = hpd_integer(n, rng)
            X = gauss_jordan_inverse(A)
            cases.append({
                "n": n,
                "A_re": [[int(z.real) for z in row] for row in A],
                "A_im": [[int(z.imag) for z in row] for row in A],
                # exact rationals as "num/den" strings
                "X_re": [[str(v[0]) for v in row] for row in X],
                "X_im": [[str(v[1]) for v in row] for row in X],
            })
    out = {
        "source": "exact Gaussian-rational Gauss-Jordan of A X = I (PAPER.md P:105-107, P:151-153)",
        "generator": "tests/golden/make_golden.py (seed 20111144)",
        "cases": cases,
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gauss_jordan.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, len(cases), "cases")


if __name__ == "__main__":
    main()
