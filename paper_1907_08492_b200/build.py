"""Build libdg_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1907_08492_b200.build [-v]

Every .cu under csrc/ is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
and linked with the host sources (g++, __float128 basis construction) against
cudart and the NCCL that torch ships (rpath'ed so the same libnccl.so.2 is used).
"""
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libdg_b200.so")
BUILD = os.path.join(ROOT, "build", "dg_b200")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nccl_dirs():
    cands = []
    try:
        import nvidia.nccl  # noqa: F401
        for p in nvidia.nccl.__path__:
            cands.append(p)
    except Exception:
        pass
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]))
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "dg.h")]
    newest_hdr = max(os.path.getmtime(h) for h in hdrs)
    objs, jobs = [], []
    common = ["-O3", "-std=c++17", "-I" + inc, "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if not force and os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(s), newest_hdr):
            continue
        if s.endswith(".cu"):
            cmd = ["nvcc", ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                   "-c", s, "-o", o] + common
        else:
            cmd = ["g++", "-fPIC", "-Wall", "-Wno-unused-function", "-c", s, "-o", o,
                   "-I/usr/local/cuda/include"] + common
        jobs.append(cmd)
    if jobs:   # independent translation units: compile in parallel
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = ["nvcc", ARCH, "-shared", "-o", OUT] + objs + [
            "-L" + lib, "-lnccl", "-lcudart", "-lquadmath", "-Xlinker", "-rpath=" + lib]
        _run(cmd, verbose)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
