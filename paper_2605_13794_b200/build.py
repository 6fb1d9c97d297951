"""Build libbgs.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo).

    python -m paper_2605_13794_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(os.path.dirname(HERE), "build", "libbgs")
LIB = os.path.join(HERE, "libbgs.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

SOURCES = ["runtime.cu", "project.cu", "sort.cu", "raster.cu", "project_bwd.cu", "route.cu", "importance.cu",
           "layout.cu", "simplify.cu", "loss.cu", "adam.cu", "densify.cu", "bucket.cu"]
# per-TU extra flags: the projection TU is pinned (no FMA contraction; IEEE div/sqrt are the
# nvcc defaults) so that integer decisions match the oracle bit for bit (D2); the
# simplification TU too (pinned fp64 ln of the race keys, R30; it also uses __d*_rn explicitly)
EXTRA = {"project.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"], "simplify.cu": ["-fmad=false"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        cands += [os.path.join(p, "nccl") for p in spec.submodule_search_locations]
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found (expected nvidia/nccl in site-packages)")


def _compile(src: str, force: bool, csrc: str = CSRC, bdir: str = BUILD) -> str:
    os.makedirs(bdir, exist_ok=True)
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    deps = [os.path.join(csrc, src), os.path.join(csrc, "bgs_internal.cuh"), os.path.join(INCLUDE, "bgs.h")]
    if not force and os.path.exists(obj) and all(os.path.getmtime(obj) >= os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "-I" + os.path.join(nccl_root(), "include"), "-I" + INCLUDE, *EXTRA.get(src, []),
           "-c", os.path.join(csrc, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(obj + ".log", "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, csrc: str = CSRC, name: str = "") -> str:
    """name != "": an A/B variant built from another source tree (e.g. a `git archive` of a
    previous commit) into build/libbgs_<name>/ and libbgs_<name>.so; bgs.py loads it when
    BGS_LIB=libbgs_<name>.so is set.  The product library is always libbgs.so."""
    bdir = BUILD + (f"_{name}" if name else "")
    lib = LIB if not name else os.path.join(HERE, f"libbgs_{name}.so")
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, csrc, bdir), SOURCES))
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(o) for o in objs):
        return lib
    nl = os.path.join(nccl_root(), "lib")
    tmp = lib + f".{os.getpid()}.tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L" + nl, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nl]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    a = sys.argv[1:]
    kw = {}
    if "--csrc" in a:
        kw["csrc"] = os.path.abspath(a[a.index("--csrc") + 1])
    if "--name" in a:
        kw["name"] = a[a.index("--name") + 1]
    print(build(force="--force" in a, **kw))
