"""Build libpqkv_sm100.so in-tree with nvcc for sm_100a.

    python -m paper_2504_03661_b200.build        # incremental
    python -m paper_2504_03661_b200.build -f     # force

The shared library lands in ``paper_2504_03661_b200/_lib/`` (git-ignored, but
shipped to the GPU box by gpurun's snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libpqkv_sm100.so")
SOURCES = ["tables.cu", "encode.cu", "decode.cu", "fileio.cu", "vstore.cu"]
HEADERS = ["common.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
    "-diag-suppress", "550",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(INCLUDE, "pqkv_sm100.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB,
          defines: tuple = ()) -> str:
    """Compile every .cu for sm_100a and link libpqkv_sm100.so; return its path.
    `defines` (e.g. ("PQKV_TRACE",)) builds a diagnostic variant into `lib`."""
    if not force and not _stale(lib):
        return lib
    out_dir = os.path.dirname(os.path.abspath(lib))
    os.makedirs(out_dir, exist_ok=True)
    # object names unique per output library, so parallel builds of variants
    # into one directory do not collide
    tag = "_" + os.path.basename(lib).replace(".", "_") + "_".join(defines)
    objs, procs = [], []
    try:
        # the translation units compile in parallel (decode.cu dominates)
        for src in SOURCES:
            obj = os.path.join(out_dir, src.replace(".cu", f"{tag}.o"))
            cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{x}" for x in defines], "-I", INCLUDE, "-c",
                   os.path.join(CSRC, src), "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            objs.append(obj)
            procs.append((src, subprocess.Popen(cmd)))
        failed = [src for src, p in procs if p.wait() != 0]
        if failed:
            raise RuntimeError(f"nvcc failed on {', '.join(failed)}")
        tmp = lib + ".tmp"
        subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-o", tmp, *objs], check=True)
        os.replace(tmp, lib)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
