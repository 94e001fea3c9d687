"""Build libvegas_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2408_09229_b200.build        # or __graft_entry__.build()

Each .cu in csrc/ is compiled separately (in parallel) with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false`` and linked
with NCCL (the torch-bundled libnccl.so.2, so one NCCL lives in the process).
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libvegas_b200.so")
# tuning variants: VPB_BUILD_DEFINES="-DVPB_FILL_NT=640" VPB_BUILD_OUT=/path/lib.so
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def nccl_paths():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (same one torch.distributed uses)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(objs) -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "vegas_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    global LIB
    extra = os.environ.get("VPB_BUILD_DEFINES", "").split()
    if os.environ.get("VPB_BUILD_OUT"):
        LIB = os.path.abspath(os.environ["VPB_BUILD_OUT"])
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(os.path.dirname(LIB), "obj" + ("_" + str(abs(hash(tuple(extra)))) if extra else ""))
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if not force and not _stale(objs):
        return LIB
    nvcc = _nvcc()
    inc, lib = nccl_paths()

    def compile_one(pair):
        src, obj = pair
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-I", inc, "-I", os.path.join(ROOT, "include"),
               "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        logs = list(ex.map(compile_one, zip(srcs, objs)))
    if verbose:
        for l in logs:
            sys.stderr.write(l)
    cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={lib}", "-cudart", "static"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
