"""CPU-only checks of the boundary: the C-ABI library loads and exports every symbol that
include/hpdinv.h declares; argument validation needs no GPU (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hpdinv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M))


@pytest.fixture(scope="module")
def lib():
    from paper_1111_4144_b200 import _build
    _build.build()
    import paper_1111_4144_b200 as hp
    return hp.lib()


def test_exports_every_declared_symbol(lib):
    import paper_1111_4144_b200 as hp
    decl = _declared()
    assert decl == set(hp.EXPORTS), decl ^ set(hp.EXPORTS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", hp._lib.LIB_PATH]).decode()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for name in decl:
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_validation_without_gpu(lib):
    z = ctypes.c_void_p(0)
    # batch == 0 is a no-op; argument errors return -k before touching the device
    assert lib.chol_inv_batched_c64(0, 8, z, 1, 0, z, 1, 0, z, z) == 0
    assert lib.ldl_inv_batched_c128(-5, 8, z, 1, 8, z, 1, 8, z, z) == -1
    assert lib.chol_inv_batched_c128(4, 0, z, 1, 8, z, 1, 8, z, z) == -2
    assert lib.ldl_inv_batched_c64(4, 65, z, 1, 8, z, 1, 8, z, z) == -2
    assert lib.chol_inv_batched_c64(4, 8, z, 1, 8, z, 1, 8, z, z) == -3
    fake = ctypes.c_void_p(1 << 20)
    assert lib.chol_inv_batched_c64(4, 8, fake, 2, 2, fake, 64, 1, fake, z) == -4
    assert lib.chol_inv_batched_c64(4, 8, fake, 1, 3, fake, 64, 1, fake, z) == -4   # ld < batch
    assert lib.chol_inv_batched_c64(4, 8, fake, 64, 1, fake, 63, 1, fake, z) == -7  # sm < n^2
    assert lib.hpdinv_kernel_name(0, 0, 1 << 20, 8, 1, 1 << 20, 1, 1 << 20) is not None
    assert lib.hpdinv_kernel_name(0, 0, 16, 65, 1, 16, 1, 16) is None
    assert lib.hpdinv_host_workspace_bytes(0, 8, 1024) >= 2 * 64 * 8 * 1024
    assert lib.hpdinv_inv_host(0, 0, 4, 8, z, 1, 4, z, 1, 4, z, z, 0, 0, z) == -5
    assert b"sm_100a" in lib.hpdinv_version()
    # batched solve (f1): same conventions, vectors interleaved or contiguous
    assert lib.chol_solve_batched_c64(0, 8, z, 1, 0, z, 1, 0, z, 1, 0, z, z) == 0
    assert lib.ldl_solve_batched_c128(-1, 8, z, 1, 8, z, 1, 8, z, 1, 8, z, z) == -1
    assert lib.chol_solve_batched_c128(4, 65, z, 1, 8, z, 1, 8, z, 1, 8, z, z) == -2
    assert lib.chol_solve_batched_c64(4, 8, z, 1, 8, z, 1, 8, z, 1, 8, z, z) == -3
    assert lib.chol_solve_batched_c64(4, 8, fake, 1, 4, z, 1, 4, z, 1, 4, z, z) == -6
    assert lib.chol_solve_batched_c64(4, 8, fake, 1, 4, fake, 2, 2, z, 1, 4, z, z) == -7
    assert lib.chol_solve_batched_c64(4, 8, fake, 1, 4, fake, 8, 1, fake, 7, 1, z, z) == -10
    assert lib.ldl_solve_batched_c64(4, 8, fake, 1, 4, fake, 8, 1, fake, 1, 4, z, z) == -12
    assert lib.hpdinv_solve_kernel_name(0, 0, 8) == b"k_solve_reg<c64,chol>"
    assert lib.hpdinv_solve_kernel_name(1, 1, 64) == b"k_solve_gen<c128,ldl>"
    assert lib.hpdinv_solve_kernel_name(0, 0, 65) is None
    assert lib.hpdinv_solve_host_workspace_bytes(0, 8, 1024) >= 2 * 8 * (64 + 16) * 1024
    assert lib.hpdinv_solve_host(0, 0, 4, 8, z, 1, 4, z, 1, 4, z, 1, 4, z, z, 0, 0, z) == -5
    assert lib.hpdinv_solve_host(2, 0, 4, 8, z, 1, 4, z, 1, 4, z, 1, 4, z, z, 0, 0, z) == -1
    # existing methods (f3): argument k of the 10-argument form is k + 2
    assert lib.hpdinv_inv_batched_method(4, 0, 4, 8, fake, 1, 4, fake, 1, 4, fake, z) == -1
    assert lib.hpdinv_inv_batched_method(2, 2, 4, 8, fake, 1, 4, fake, 1, 4, fake, z) == -2
    assert lib.hpdinv_inv_batched_method(2, 0, -1, 8, fake, 1, 4, fake, 1, 4, fake, z) == -3
    assert lib.hpdinv_inv_batched_method(3, 1, 4, 0, fake, 1, 4, fake, 1, 4, fake, z) == -4
    assert lib.hpdinv_inv_batched_method(0, 0, 4, 8, z, 1, 4, fake, 1, 4, fake, z) == -5
    assert lib.hpdinv_inv_batched_method(2, 0, 0, 8, z, 1, 4, z, 1, 4, z, z) == 0
    assert lib.hpdinv_method_kernel_name(2, 0, 8) == b"k_base_reg<c64,eqsolve>"
    assert lib.hpdinv_method_kernel_name(3, 1, 33) == b"k_base_gen<c128,trimat>"
    assert lib.hpdinv_method_kernel_name(0, 0, 8) is None
    # non-Hermitian inversion (f2): the 10-argument convention
    assert lib.nonherm_inv_batched_c64(0, 8, z, 1, 0, z, 1, 0, z, z) == 0
    assert lib.nonherm_inv_batched_c128(4, 0, fake, 1, 4, fake, 1, 4, fake, z) == -2
    assert lib.nonherm_inv_batched_c64(4, 8, fake, 2, 2, fake, 1, 4, fake, z) == -4
    assert lib.nonherm_inv_batched_c64(4, 8, fake, 1, 4, fake, 1, 4, z, z) == -9
    assert lib.hpdinv_nonherm_kernel_name(0, 8) == b"k_nh_reg<c64>"
    assert lib.hpdinv_nonherm_kernel_name(1, 8) == b"k_nh_gen<c128>"
    # fixed-point emulation (f4)
    assert lib.hpdinv_fxp_inv_batched(3, 4, 11, 4, 8, fake, fake, fake, fake, z) == -1
    assert lib.hpdinv_fxp_inv_batched(0, 30, 11, 4, 8, fake, fake, fake, fake, z) == -2
    assert lib.hpdinv_fxp_inv_batched(0, 4, 11, -1, 8, fake, fake, fake, fake, z) == -4
    assert lib.hpdinv_fxp_inv_batched(0, 4, 11, 4, 17, fake, fake, fake, fake, z) == -5
    assert lib.hpdinv_fxp_inv_batched(0, 4, 11, 4, 8, z, fake, fake, fake, z) == -6
    assert lib.hpdinv_fxp_inv_batched(1, 4, 11, 0, 8, z, z, z, z, z) == 0


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle and refuses CPU tensors."""
    pkg = os.path.join(ROOT, "paper_1111_4144_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
    import torch
    import paper_1111_4144_b200 as hp
    with pytest.raises(ValueError):
        hp.chol_inv_batched_c64(torch.zeros(2, 4, 4, dtype=torch.complex64))
