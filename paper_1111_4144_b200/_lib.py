"""ctypes loader for the in-tree libhpdinv.so (include/hpdinv.h).  Fails loudly if the CUDA
library has not been built: there is no CPU fallback anywhere in the product path."""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPDINV_LIB") or os.path.join(HERE, "libhpdinv.so")   # override: A/B builds

_lib = None


class HpdinvError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HpdinvError(
            "libhpdinv.so is not built (%s). Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `python paper_1111_4144_b200/_build.py`." % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    inv_args = [I64, I, P, I64, I64, P, I64, I64, P, P]
    for name in ("chol_inv_batched_c64", "chol_inv_batched_c128",
                 "ldl_inv_batched_c64", "ldl_inv_batched_c128"):
        f = getattr(L, name)
        f.restype = I
        f.argtypes = inv_args
    solve_args = [I64, I, P, I64, I64, P, I64, I64, P, I64, I64, P, P]
    for name in ("chol_solve_batched_c64", "chol_solve_batched_c128",
                 "ldl_solve_batched_c64", "ldl_solve_batched_c128"):
        f = getattr(L, name)
        f.restype = I
        f.argtypes = solve_args
    for name in ("nonherm_inv_batched_c64", "nonherm_inv_batched_c128"):
        f = getattr(L, name)
        f.restype = I
        f.argtypes = inv_args
    L.hpdinv_nonherm_kernel_name.restype = ctypes.c_char_p
    L.hpdinv_nonherm_kernel_name.argtypes = [I, I]
    L.hpdinv_fxp_inv_batched.restype = I
    L.hpdinv_fxp_inv_batched.argtypes = [I, I, I, I64, I, P, P, P, P, P]
    L.hpdinv_inv_batched_method.restype = I
    L.hpdinv_inv_batched_method.argtypes = [I, I] + inv_args
    L.hpdinv_method_kernel_name.restype = ctypes.c_char_p
    L.hpdinv_method_kernel_name.argtypes = [I, I, I]
    L.hpdinv_solve_host_workspace_bytes.restype = ctypes.c_size_t
    L.hpdinv_solve_host_workspace_bytes.argtypes = [I, I, I64]
    L.hpdinv_solve_host.restype = I
    L.hpdinv_solve_host.argtypes = [I, I, I64, I, P, I64, I64, P, I64, I64, P, I64, I64, P, P,
                                    ctypes.c_size_t, I64, P]
    L.hpdinv_solve_kernel_name.restype = ctypes.c_char_p
    L.hpdinv_solve_kernel_name.argtypes = [I, I, I]
    L.hpdinv_host_workspace_bytes.restype = ctypes.c_size_t
    L.hpdinv_host_workspace_bytes.argtypes = [I, I, I64]
    L.hpdinv_inv_host.restype = I
    L.hpdinv_inv_host.argtypes = [I, I, I64, I, P, I64, I64, P, I64, I64, P, P, ctypes.c_size_t,
                                  I64, P]
    L.hpdinv_kernel_name.restype = ctypes.c_char_p
    L.hpdinv_kernel_name.argtypes = [I, I, I64, I, I64, I64, I64, I64]
    L.hpdinv_version.restype = ctypes.c_char_p
    L.hpdinv_version.argtypes = []
    _lib = L
    return L


# Every symbol include/hpdinv.h declares (checked by tests/test_abi.py without a GPU).
EXPORTS = (
    "chol_inv_batched_c64", "chol_inv_batched_c128",
    "ldl_inv_batched_c64", "ldl_inv_batched_c128",
    "chol_solve_batched_c64", "chol_solve_batched_c128",
    "ldl_solve_batched_c64", "ldl_solve_batched_c128", "hpdinv_solve_kernel_name",
    "hpdinv_solve_host_workspace_bytes", "hpdinv_solve_host",
    "hpdinv_inv_batched_method", "hpdinv_method_kernel_name",
    "nonherm_inv_batched_c64", "nonherm_inv_batched_c128", "hpdinv_nonherm_kernel_name",
    "hpdinv_fxp_inv_batched",
    "hpdinv_host_workspace_bytes", "hpdinv_inv_host",
    "hpdinv_kernel_name", "hpdinv_version",
)
