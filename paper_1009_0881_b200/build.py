"""In-tree build of the sm_100a extension: paper_1009_0881_b200/_lib/libmlnmf_b200.so.

Plain nvcc (no torch extension machinery): every CUDA translation unit is
compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``; the
CUDA runtime is linked statically and NCCL is dlopen'ed at run time, so the
shared object only depends on libc/libstdc++/libdl.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libmlnmf_b200.so")
REPO = os.path.dirname(HERE)

SOURCES = ["engine.cu", "ix_gemm.cu", "hals_reg.cu", "restrict_tma.cu", "gram_dmma.cu", "hals_dmma.cu", "scheduler.cpp", "capi.cpp", "host_io.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CLI_SOURCES = ["cli_main.cpp"]  # dataset / result I/O from the library (host_io.cpp)
CLI = os.path.join(OUT_DIR, "mlnmf_b200")  # the CLI executable (reference: tools/mlnmf_main.cpp)


def _nccl_paths():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (headers + lib)
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
    except Exception:
        base = None
    inc = os.path.join(base, "include") if base else "/usr/include"
    lib = os.path.join(base, "lib", "libnccl.so.2") if base else "/usr/lib/x86_64-linux-gnu/libnccl.so.2"
    return inc, lib


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _flags():
    inc, lib = _nccl_paths()
    return ARCH + [
        "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v" if os.environ.get("MLB_PTXAS_V") else "-O3",
        f"-I{inc}", f"-I{os.path.join(REPO, 'include')}", f'-DMLB_NCCL_PATH="{lib}"',
        "--expt-relaxed-constexpr",
    ]


def _deps(src):
    # every TU depends on every header in csrc/ and include/ (small project)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hdrs.append(os.path.join(REPO, "include", "mlnmf_b200.h"))
    return [src] + hdrs + [__file__]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = _nvcc()
    flags = _flags()
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OUT_DIR, s + ".o")
        objs.append(obj)
        if force or _stale(obj, _deps(src)):
            lang = ["-x", "cu"] if s.endswith(".cu") else ["-x", "c++"]
            jobs.append([nvcc] + flags + lang + ["-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        if verbose and (p.stdout or p.stderr):
            print(p.stdout, p.stderr, flush=True)

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([nvcc] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lpthread", "-lrt"])
    # the CLI front-end (host C++ over the C-ABI); no -march and no fp
    # contraction, so the synth generator rounds like the reference build
    cli_src = [os.path.join(CSRC, s) for s in CLI_SOURCES]
    if force or _stale(CLI, cli_src + _deps(cli_src[0]) + [LIB]):
        run([os.environ.get("MLB_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"), "-std=c++20", "-O2", "-ffp-contract=off", "-Wall",
             f"-I{os.path.join(REPO, 'include')}", f"-I{CSRC}", "-o", CLI] + cli_src +
            [f"-L{OUT_DIR}", "-lmlnmf_b200", "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
