"""Build libdeepthin_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1802_06944_b200.build [--force] [--timing]

The shared library lands next to this file (``_lib/libdeepthin_b200.so``) so
it travels with the repository snapshot to the GPU box.

``--timing`` builds a separate diagnostics library (``_lib/libdeepthin_b200_timing.so``,
loaded only with ``DEEPTHIN_LIB=<path>``) compiled with ``-DDEEPTHIN_TIMING_SWITCHES``: the only
build that reads the DEEPTHIN_DBG_* / *_TRACE timing-experiment switches. The product library
never contains them.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUTDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUTDIR, "libdeepthin_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
              "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build the sm_100a kernels")
    return cand


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _fingerprint(extra=()) -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)) + ["../../include/deepthin_b200.h"]:
        path = os.path.join(CSRC, name)
        if os.path.isfile(path):
            h.update(name.encode())
            with open(path, "rb") as f:
                h.update(f.read())
    h.update(" ".join(ARCH + NVCC_FLAGS + list(extra)).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, timing: bool = False) -> str:
    os.makedirs(OUTDIR, exist_ok=True)
    extra = ["-DDEEPTHIN_TIMING_SWITCHES"] if timing else []
    if os.environ.get("DEEPTHIN_TEST_WAIT", "0") not in ("", "0"):
        extra.append("-DDEEPTHIN_TEST_WAIT")  # experiment: non-blocking mbarrier.test_wait polls
    if os.environ.get("DEEPTHIN_BOUNDED_WAITS", "0") not in ("", "0"):
        extra.append("-DDEEPTHIN_BOUNDED_WAITS")  # trap on an mbarrier protocol bug (slower waits)
    lib = LIB.replace(".so", "_timing.so") if timing else LIB
    stamp = os.path.join(OUTDIR, "build_timing.stamp" if timing else "build.stamp")
    fp = _fingerprint(extra)
    if not force and os.path.exists(lib) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == fp:
                return lib
    cc = nvcc()
    objs = []

    def compile_one(src):
        obj = os.path.join(OUTDIR, src.replace(".cu", "_t.o" if timing else ".o"))
        cmd = [cc, *ARCH, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + ".tmp"
    r = subprocess.run([cc, *ARCH, "-shared", "-o", tmp, *objs,
                        "-Xlinker", "-rpath,/usr/local/cuda/lib64"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    with open(stamp, "w") as f:
        f.write(fp)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timing="--timing" in sys.argv))
