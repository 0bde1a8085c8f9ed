"""Build libkcore_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2512_00233_b200.build          # incremental
    python -m paper_2512_00233_b200.build --force

The library is the drop-in C-ABI declared in include/kcore_b200.h.  It is
built in-tree so the .so travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libkcore_b200.so")
SOURCES = ["kc_solve.cu", "kc_count.cu", "kc_count_split.cu", "kc_tail.cu", "kc_peel.cu", "kc_prep.cu", "kc_api.cu", "kc_gen.cu", "kc_ingest.cu", "kc_stage.cu", "kc_hostcopy.cpp"]
HEADERS = ["kc_internal.h", "kc_dev.cuh", "kc_count_impl.cuh", os.path.join("..", "..", "include", "kcore_b200.h")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-Wno-deprecated-declarations",
    "-Xptxas", "-warn-spills",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB,
          build_dir: str = BUILD) -> str:
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc()] + FLAGS + [f"-D{d}" for d in defines] + ["-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, r in zip(jobs, results):
            if verbose and (r.stdout or r.stderr):
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if force or jobs or _stale(lib, objs):
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib] + objs + \
              ["-Xcompiler", "-fPIC", "-cudart", "static", "-lz"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[],
                    help="extra preprocessor define (A/B development builds)")
    ap.add_argument("--variant", default="", help="build libkcore_b200_<variant>.so")
    a = ap.parse_args()
    if a.variant:
        print(build(force=a.force, verbose=a.verbose, defines=a.defines,
                    lib=os.path.join(HERE, f"libkcore_b200_{a.variant}.so"),
                    build_dir=os.path.join(BUILD, a.variant)))
    else:
        print(build(force=a.force, verbose=a.verbose, defines=a.defines))
