"""In-tree build of the native components (no JIT cache: the .so / binaries
travel to the GPU box inside the repo snapshot).

  lib/libtaichi_b200.so   CUDA library (sm_100a): kernels + the C ABI of include/taichi_b200.h
  lib/taichi_sim          host engine CLI (C++20, include/pdsim)
  lib/reftests/<t>        the reference's own gtest files compiled against include/pdsim
                          (drop-in check; GoogleTest replaced by oracle/gtest_shim)

Host C++ is compiled with -O2 -ffp-contract=off (FMA contraction
changes the double-precision logical clock and therefore schedules).
"""
from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
REPO = PKG.parent
LIB = PKG / "lib"
CSRC = PKG / "csrc"
INCLUDE = REPO / "include"
NLOHMANN = pathlib.Path(
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
REF_TESTS = ["cost_model_test", "cluster_test", "proxy_test", "decode_flow_test",
             "metrics_test", "workload_test", "engine_test"]
HOST_FLAGS = ["-std=c++20", "-O2", "-ffp-contract=off"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared"]


def _stale(target: pathlib.Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(pathlib.Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, **kw):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True, **kw)


def build_cuda(force: bool = False) -> pathlib.Path:
    out = LIB / "libtaichi_b200.so"
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "taichi_b200.h"]
    if force or _stale(out, deps):
        LIB.mkdir(exist_ok=True)
        tmp = out.with_suffix(".so.tmp")
        _run([NVCC, *NVCC_FLAGS, f"-I{INCLUDE}", CSRC / "taichi_b200.cu", "-o", tmp])
        tmp.replace(out)
    return out


def build_host(force: bool = False) -> pathlib.Path:
    out = LIB / "taichi_sim"
    deps = list((INCLUDE / "pdsim").glob("*.hpp")) + list((INCLUDE / "taichi").glob("*.hpp")) + \
        [CSRC / "taichi_sim.cpp"]
    if force or _stale(out, deps):
        LIB.mkdir(exist_ok=True)
        _run([CXX, *HOST_FLAGS, "-Wall", "-Wextra", f"-I{INCLUDE}", f"-I{NLOHMANN}",
              CSRC / "taichi_sim.cpp", "-o", out, "-pthread"])
    return out


def build_cuda_variant(name: str, defines: list[str]) -> pathlib.Path:
    """Extra library builds for A/B microbenchmarks (e.g. TC_GEMM_BK=64); not used by the product."""
    out = LIB / f"libtaichi_b200_{name}.so"
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "taichi_b200.h"]
    if _stale(out, deps):
        _run([NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{INCLUDE}", CSRC / "taichi_b200.cu", "-o", out])
    return out


def build_serve(force: bool = False) -> pathlib.Path:
    """Host engine + GPU executor, linked against lib/libtaichi_b200.so (rpath $ORIGIN)."""
    out = LIB / "taichi_serve"
    so = build_cuda(force)
    deps = list((INCLUDE / "pdsim").glob("*.hpp")) + list((INCLUDE / "taichi").glob("*.hpp")) + \
        [CSRC / "taichi_serve.cpp", INCLUDE / "taichi_b200.h", so]
    if force or _stale(out, deps):
        _run([CXX, *HOST_FLAGS, "-Wall", "-Wextra", f"-I{INCLUDE}", f"-I{NLOHMANN}", CSRC / "taichi_serve.cpp",
              "-o", out, f"-L{LIB}", "-ltaichi_b200", "-Wl,-rpath,$ORIGIN", "-pthread"])
    return out


def build_reftests(force: bool = False) -> list[pathlib.Path]:
    """Reference gtest sources (read from /root/reference, never copied) vs our headers."""
    src_dir = pathlib.Path("/root/reference/proj/tests")
    outs = []
    if not src_dir.exists():
        return [LIB / "reftests" / t for t in REF_TESTS if (LIB / "reftests" / t).exists()]
    shim = REPO / "oracle" / "gtest_shim"
    (LIB / "reftests").mkdir(parents=True, exist_ok=True)
    main_o = LIB / "reftests" / "gtest_main.o"
    if force or _stale(main_o, [shim / "gtest_main.cpp", shim / "gtest" / "gtest.h"]):
        _run([CXX, *HOST_FLAGS, f"-I{shim}", "-c", shim / "gtest_main.cpp", "-o", main_o])
    hdrs = list((INCLUDE / "pdsim").glob("*.hpp")) + [shim / "gtest" / "gtest.h", main_o]
    procs = []
    for t in REF_TESTS:
        out = LIB / "reftests" / t
        outs.append(out)
        if force or _stale(out, hdrs + [src_dir / f"{t}.cpp"]):
            cmd = [CXX, *HOST_FLAGS, "-w", f"-I{shim}", f"-I{INCLUDE}", f"-I{NLOHMANN}",
                   src_dir / f"{t}.cpp", main_o, "-o", out, "-pthread"]
            print("+", " ".join(map(str, cmd)), flush=True)
            procs.append(subprocess.Popen([str(c) for c in cmd]))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("reference test build failed")
    return outs


def build_oracle() -> None:
    """Compile the checker (oracle/_ref) when the reference tree is present."""
    if pathlib.Path("/root/reference/proj/include/pdsim").exists() and shutil.which("make"):
        _run(["make", "-C", REPO / "oracle", "-j8"])


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_host(force)
    build_serve(force)
    build_reftests(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
