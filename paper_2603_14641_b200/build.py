"""In-tree build of libqsr.so (sm_100a) — no JIT cache, the .so travels with the repo snapshot.

    python paper_2603_14641_b200/build.py          # incremental
    python paper_2603_14641_b200/build.py --force
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "_obj"
LIB = PKG / "libqsr.so"
CLI_SRC = PKG / "cli" / "quasar_cli.cpp"
CLI = PKG / "bin" / "quasar"   # the reference CLI (tools/quasar.cpp) on this engine
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", str(PKG.parent / "include")]
SOURCES = ["host_circuit.cpp", "capi.cpp", "engine.cpp", "k_gates.cu", "k_transpose.cu", "k_measure.cu", "k_batch.cu",
           "k_frames.cu", "exchange.cu", "shard.cpp", "stream.cpp", "fuse.cpp", "qasm.cpp", "k_validity.cu"]
HEADERS = ["host.hpp", "device.hpp", "common.cuh", "abi.hpp", "engine.hpp", "exchange.hpp", "fuse.hpp", "stream_plan.hpp"]


def _newest_header() -> float:
    hs = [CSRC / h for h in HEADERS] + [PKG.parent / "include" / "qsr.h"]
    return max(h.stat().st_mtime for h in hs)


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    hdr = _newest_header()
    objs = []
    for src in SOURCES:
        sp = CSRC / src
        op = OBJ / (src + ".o")
        objs.append(op)
        if not force and op.exists() and op.stat().st_mtime >= max(sp.stat().st_mtime, hdr):
            continue
        cmd = [NVCC, *ARCH, *COMMON, "-c", str(sp), "-o", str(op)]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-I", str(PKG.parent / "include"),
                   "-I", "/usr/local/cuda/include", "-c", str(sp), "-o", str(op)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    CLI.parent.mkdir(exist_ok=True)
    if force or not CLI.exists() or CLI.stat().st_mtime < max(LIB.stat().st_mtime, CLI_SRC.stat().st_mtime):
        cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-I", str(PKG.parent / "include"), str(CLI_SRC), "-o", str(CLI),
               "-L", str(PKG), "-lqsr", "-Wl,-rpath,$ORIGIN/..", "-pthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
