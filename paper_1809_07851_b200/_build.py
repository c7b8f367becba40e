"""Build the fastconv CUDA library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfastconv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "fastconv.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str | None = None) -> str:
    """Compile every .cu to an object in parallel (one nvcc per translation unit), then
    link the shared library.  extra_flags / out: experiment builds (A/B variants) into
    another library path; the product library is LIB, built with no extra flags."""
    target = out or LIB
    if not force and out is None and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build") if out is None else target + ".objs"
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared",)] + list(extra_flags)
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append((src, obj, [NVCC] + compile_flags + ["-c", "-o", obj, src]))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[2], capture_output=True, text=True), jobs))
    log = os.path.join(PKG, "build.log")
    tmp = target + ".tmp"
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", tmp] + \
        [j[1] for j in jobs] + ["-lcuda"] * 0
    with open(log, "w") as f:
        for (src, obj, cmd), res in zip(jobs, results):
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        bad = [(j, r) for j, r in zip(jobs, results) if r.returncode != 0]
        if bad:
            raise RuntimeError("nvcc failed (see %s):\n%s" % (log, "\n".join(r.stderr[-3000:] for _, r in bad)))
        res = subprocess.run(link, capture_output=True, text=True)
        f.write(" ".join(link) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("link failed (see %s):\n%s" % (log, res.stderr[-4000:]))
    if verbose:
        print("".join(r.stderr for r in results))
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
