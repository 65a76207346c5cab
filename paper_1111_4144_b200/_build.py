"""Builds libhpdinv.so in-tree with nvcc for sm_100a (static cudart, -lineinfo).

One object per csrc/*.cu (compiled in parallel), linked into a shared library."""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhpdinv.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return (glob.glob(os.path.join(HERE, "csrc", "*.cu*")) + glob.glob(os.path.join(HERE, "csrc", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _compile(src, verbose, extra=(), objdir=None):
    objdir = objdir or OBJ
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps() if not d.endswith(".cu") or d == src):
        return obj
    cmd = [NVCC] + CFLAGS + list(extra) + ["-c", src, "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr))
    if verbose and r.stderr.strip():
        print(r.stderr.strip())
    os.replace(obj + ".tmp", obj)
    return obj


def build(force=False, verbose=False, lib=LIB, extra=(), objdir=None):
    """Build `lib` (default: the in-tree libhpdinv.so).  `extra` nvcc flags (e.g. a -D for an
    A/B variant) go with their own object directory."""
    objdir = objdir or OBJ
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(s) for s in deps()):
        return lib
    os.makedirs(objdir, exist_ok=True)
    if force:
        for o in glob.glob(os.path.join(objdir, "*.o")):
            os.remove(o)
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, extra, objdir), sources()))
    tmp = lib + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    if "--variant" in sys.argv:      # e.g. --variant noffma2 -DHPDINV_NO_FFMA2
        i = sys.argv.index("--variant")
        name, flags = sys.argv[i + 1], sys.argv[i + 2:]
        out = build(force="--force" in sys.argv, verbose=True, lib=os.path.join(HERE, "libhpdinv_%s.so" % name),
                    extra=[f for f in flags if f != "--force"], objdir=os.path.join(OBJ, name))
        print("built", out)
    else:
        build(force="--force" in sys.argv, verbose=True)
        print("built", LIB)
