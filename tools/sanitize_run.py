#!/usr/bin/env python
"""Small launches of every kernel family, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

k_reg (n = 4, 8 c64; n = 6 c128), k_grp (n = 16, 32 c64), k_lane (n = 20 c64, n = 12 c128),
k_generic (n = 48 c64), k_blk (n = 32 c128, n = 64 c128 LDL, n = 64 c64), k_dmma (n = 64 c128
Cholesky, AoS A), the solves, the non-Hermitian kernels, the existing methods and the
fixed-point emulation.  Each call's info/X is checked loosely (finite, info == 0) so a run
that silently did nothing is visible too."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1111_4144_b200 as hp  # noqa: E402
from paper_1111_4144_b200 import workloads as wl  # noqa: E402


def gen(n, dtype, batch, kind="bbh", task="inv"):
    cfg = wl.Config(90, n, dtype, 0, "chol", "aos", kind, float(n), 0.1 if kind == "bbh" else 1.0, task=task)
    if kind == "nonherm":
        cfg = wl.Config(91, n, dtype, 0, "chol", "aos", "nonherm", 2.0 * n ** 0.5, 1.0, task="nonherm")
    return wl.generate(cfg, 0, batch, device="cuda")


def check(name, X, info):
    torch.cuda.synchronize()
    ok = bool((info == 0).all()) and bool(torch.isfinite(torch.view_as_real(X)).all())
    print("%-34s %s" % (name, "ok" if ok else "CHECK"), flush=True)


def main():
    c64, c128 = torch.complex64, torch.complex128
    cases = [(4, c64, "soa"), (8, c64, "soa"), (6, c128, "aos"), (16, c64, "soa"), (32, c64, "aos"),
             (20, c64, "aos"), (12, c128, "aos"), (48, c64, "aos"), (32, c128, "aos"), (64, c64, "aos"),
             (64, c128, "aos")]
    for n, dt, layout in cases:
        A = gen(n, dt, 67 if n <= 32 else 13)
        _, view = wl.to_layout(A, layout)
        for method in ("chol", "ldl"):
            X, info = hp.invert(view, method)
            check("inv n=%d %s %s %s [%s]" % (n, dt, method, layout,
                                              hp.kernel_name(method, dt, A.shape[0], n, (view.stride(0), view.stride(2)))),
                  X, info)
    for n, dt in ((8, c64), (16, c64), (6, c128)):
        A = gen(n, dt, 65)
        Y = torch.randn(65, n, dtype=dt, device="cuda")
        for method in ("chol", "ldl"):
            Xv, info = hp.solve(A, Y, method)
            check("solve n=%d %s %s" % (n, dt, method), Xv, info)
    for n, dt in ((8, c64), (12, c64), (6, c128)):
        D = gen(n, dt, 65, kind="nonherm")
        Y, info = hp.invert_nonhermitian(D)
        check("nonherm n=%d %s" % (n, dt), Y, info)
    for method in ("eqsolve", "trimat"):
        for n, dt in ((8, c64), (12, c64)):
            A = gen(n, dt, 65)
            X, info = hp.invert_method(A, method)
            check("%s n=%d %s" % (method, n, dt), X, info)
    cfg8 = wl.CONFIGS[8]
    _, raw = wl.generate_fxp(cfg8, 0, 64, device="cuda")
    X, info, nsat = hp.fxp_invert(raw, cfg8.qm, cfg8.qf, "proposed")
    torch.cuda.synchronize()
    print("%-34s %s" % ("fxp n=16", "ok" if bool((info == 0).all()) else "CHECK"), flush=True)
    print("SANITIZE_RUN_DONE", flush=True)


if __name__ == "__main__":
    main()
