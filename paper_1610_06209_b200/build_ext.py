"""Build the sm_100a extension in-tree: paper_1610_06209_b200/_lib/libspinners_b200.so.

Each translation unit is compiled by its own nvcc process (in parallel), then
linked into one shared library that exports only the C ABI of
include/spinners_b200.h.  `python paper_1610_06209_b200/build_ext.py` (or
`__graft_entry__.build()`) rebuilds when any source is newer than the library;
`--force` recompiles every translation unit.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(PKG, "_lib", "obj")
LIB = os.path.join(LIBDIR, "libspinners_b200.so")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(ROOT, "include", "spinners_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def _compile(src: str, objdir: str = OBJDIR, extra: tuple = (), force: bool = False) -> str:
    obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
    hdr_t = max(os.path.getmtime(d) for d in _deps() if not d.endswith(".cu"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
        return obj
    cmd = [NVCC] + FLAGS + list(extra) + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True, variant: str = "", defines: tuple = ()) -> str:
    """Build the library.  A named variant (A/B experiments: extra -D flags) goes to
    _lib/variants/<name>/ and is loaded by setting SPN_LIB to its path."""
    lib, objdir = LIB, OBJDIR
    if variant:
        lib = os.path.join(LIBDIR, "variants", variant, "libspinners_b200.so")
        objdir = os.path.join(LIBDIR, "variants", variant, "obj")
    elif not force and up_to_date():
        return LIB
    os.makedirs(objdir, exist_ok=True)
    srcs = _sources()
    extra = tuple("-D" + d for d in defines)
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda f: _compile(f, objdir, extra, force), srcs))
    cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcublas"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    build(force=a.force, variant=a.variant, defines=tuple(a.defines))
