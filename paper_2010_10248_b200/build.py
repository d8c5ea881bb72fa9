"""In-tree build of libstb200.so (sm_100a) with nvcc.

``python -m paper_2010_10248_b200.build`` (or ``__graft_entry__.build()``)
compiles every ``csrc/*.cu`` for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` and links them into ``paper_2010_10248_b200/libstb200.so``
(cudart linked statically, so the library has no runtime path dependency on
the toolkit).  Objects are rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libstb200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills", *ARCH, f"-I{INCLUDE}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libstb200")


def _newest_header() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    paths.append(os.path.join(INCLUDE, "stb200.h"))
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, obj: str, extra: list[str]) -> str:
    cmd = [nvcc(), "-c", src, "-o", obj, *NVCC_FLAGS, *extra]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{res.stderr[-6000:]}")
    return res.stderr


def build(verbose: bool = False, force: bool = False, extra: list[str] | None = None) -> str:
    """Compile and link; returns the library path."""
    extra = extra or []
    os.makedirs(OBJ, exist_ok=True)
    # objects built with other flags (A/B -D switches) are stale: the flag set
    # is stamped next to them and a change forces a full rebuild
    stamp = os.path.join(OBJ, "flags.stamp")
    flags = " ".join(NVCC_FLAGS + list(extra))
    old = open(stamp).read() if os.path.exists(stamp) else None
    if old != flags:
        force = True
    sources = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    hdr = _newest_header()
    jobs = []
    objs = []
    for f in sources:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), hdr):
            jobs.append((src, obj))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = {ex.submit(_compile, s, o, extra): s for s, o in jobs}
            for fut in cf.as_completed(futs):
                log = fut.result()
                if verbose and log.strip():
                    print(f"[{os.path.basename(futs[fut])}]\n{log}", file=sys.stderr)
    if jobs or force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(o) for o in objs):
        tmp = LIB + ".tmp"
        cmd = [nvcc(), "-shared", *ARCH, "-cudart", "static", "-o", tmp, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
        os.replace(tmp, LIB)
    if old != flags:
        with open(stamp, "w") as fh:
            fh.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
