"""Build liblfe.so (the product) and liblfe_test.so (test-only entry points,
linked against liblfe.so) in-tree with nvcc for sm_100a -- no JIT cache, no
torch types.  Every .cu compiles to an object in parallel, then one link per
library."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
TEST_SRC = os.path.join(CSRC, "test")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "liblfe.so")
TEST_LIB = os.path.join(PKG, "liblfe_test.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
          "-I", INCLUDE, "-I", CSRC]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def test_sources():
    return sorted(glob.glob(os.path.join(TEST_SRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def _newer(target, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(f) <= t for f in deps)


def up_to_date() -> bool:
    deps = sources() + test_sources() + headers()
    return _newer(LIB, deps) and _newer(TEST_LIB, deps)


def _compile(src: str):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    res = subprocess.run([_nvcc(), *CFLAGS, "-c", "-o", obj, src], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n" + res.stdout + res.stderr)
    return obj, res.stdout + res.stderr


def _link(out: str, objs, extra=()):
    tmp = out + f".tmp{os.getpid()}"
    res = subprocess.run([_nvcc(), *ARCH, "-shared", "-o", tmp, *objs, *extra], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link of {out} failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs, tsrcs = sources(), test_sources()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs) + len(tsrcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(_compile, srcs + tsrcs))
    logs = "".join(log for _, log in results)
    objs = [o for o, _ in results]
    _link(LIB, objs[:len(srcs)])
    # the test library resolves the host core from liblfe.so (found next to it)
    _link(TEST_LIB, objs[len(srcs):], ["-L", PKG, "-llfe", "-Xlinker", "-rpath,$ORIGIN"])
    if verbose:
        print(logs)
    with open(os.path.join(PKG, "liblfe.ptxas.txt"), "w") as f:
        f.write(logs)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
