"""Build libdock.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdock.so")
SOURCES = ["kernels.cu", "prep.cpp", "dock_abi.cpp", "screen.cpp", "cluster.cu", "results.cpp"]
HEADERS = ["dock_internal.h", "engine.h", "kernels.cuh", "philox.cuh", "prep.h", "score.cuh", "cluster.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-diag-suppress", "177"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "dock.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libdock.so (or, for experiments, a variant with extra -D defines at `out`)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    obj_dir = os.path.join(ROOT, "build", "obj" if out is None else "obj_" + os.path.basename(out))
    os.makedirs(obj_dir, exist_ok=True)
    procs, objs = [], []
    # kernels.cu is compiled once per scoring function -- D5 (dk::d5) and, with -DDK_AD4,
    # the NEXT-2 AutoDock4.1-calibrated variant (dk::ad4) -- and per part (DK_PART 1: eval /
    # init / GA / misc, 2: ADADELTA, 3: Solis-Wets, 4: the Solis-Wets parity-hook
    # instantiations; each part instantiates only its own
    # kernels).  All objects build in parallel.
    units = [(src, src + ".o", ()) for src in SOURCES if src != "kernels.cu"]
    for sf, tag in (((), "d5"), (("DK_AD4",), "ad4")):
        for part in (1, 2, 3, 4):
            units.append(("kernels.cu", f"kernels_{tag}_p{part}.cu.o", (*sf, f"DK_PART={part}")))
    for src, oname, extra in units:
        obj = os.path.join(obj_dir, oname)
        objs.append(obj)
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in (*defines, *extra)], "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode(errors="replace"))
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out.decode(errors="replace"))
    tmp = lib + f".{os.getpid()}.tmp"
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    subprocess.check_call([NVCC, *FLAGS, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
