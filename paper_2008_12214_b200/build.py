"""Build the sm_100a shared library in-tree (libhologen_b200.so).

Each csrc/*.cu translation unit is compiled in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked
into ``paper_2008_12214_b200/libhologen_b200.so``.  No torch involvement;
cudart is linked statically so the library only needs the driver.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(PKG, "libhologen_b200.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
                "-Xptxas", "-v"]

HOST_FLAGS = ["-Xcompiler", "-mpclmul"]  # host-only translation units (mtjump.cpp)


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int | None = None, defines: list[str] | None = None,
          out: str | None = None, objdir: str | None = None) -> str:
    """defines/out/objdir: tuning variants (e.g. -DHG_ROWQ_MINB=1) built beside the default library."""
    global OBJ, LIB
    if out:
        LIB, OBJ = out, objdir or out + ".obj"
    extra = [f"-D{d}" for d in (defines or [])]
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(PKG, "..", "include", "*.h"))
    objs, todo = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.splitext(os.path.basename(s))[0] + ".o")
        objs.append(o)
        if _stale(o, [s, *headers, __file__]):
            todo.append((s, o))

    def compile_one(so):
        s, o = so
        host = HOST_FLAGS if s.endswith(".cpp") else []
        cmd = [NVCC, *FLAGS, *host, *extra, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(o + ".log", "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {os.path.basename(s)}:\n{r.stderr[-4000:]}")
        return s

    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            for s in ex.map(compile_one, todo):
                if verbose:
                    print("compiled", os.path.basename(s), flush=True)
    if todo or not os.path.exists(LIB) or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lz"]  # zlib: PNG files (io_hgf.cpp)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        if verbose:
            print("linked", LIB, flush=True)
    return LIB


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("-D", action="append", default=[])
    ap.add_argument("--out")
    a = ap.parse_args()
    build(verbose=True, defines=a.D, out=a.out)
    sys.exit(0)
