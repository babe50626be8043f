"""Build the native libraries in-tree for sm_100a (no GPU needed: nvcc cross-compiles).

    python -m paper_2605_28053_b200.build_native [--force]

Outputs:
  paper_2605_28053_b200/lib/libtttstate.so   the product: C-ABI + pool + planner + kernels
  paper_2605_28053_b200/lib/libttt_gen.so    seeded input generator (bench/tests only)
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib")
OBJ = os.path.join(HERE, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", f"-I{ROOT}/include", f"-I{CSRC}"]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", f"-I{ROOT}/include", f"-I{CSRC}",
            "-I/usr/local/cuda/include"]

PRODUCT_CU = ["kernels/read_decode.cu", "kernels/read_decode_tc.cu", "kernels/write_simt.cu", "kernels/write_tc.cu",
              "kernels/read_chunk_tc.cu", "kernels/read_chunk_wide.cu", "kernels/lowrank.cu", "kernels/lowrank_tc.cu", "kernels/control.cu"]
PRODUCT_CPP = ["tttstate.cpp", "planner.cpp"]
GEN_CU = ["gen/ttt_gen.cu"]


def _headers():
    hs = []
    for d, _, fs in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in fs if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "tttstate.h"))
    return hs


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, force, log):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace("/", "_") + ".o")
    if not force and not _stale(obj, [path] + _headers()):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", path, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append((src, r.stdout + r.stderr))
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    return obj


def _link(objs, out, force):
    if not force and not _stale(out, objs):
        return
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs + ["-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {out}\n{r.stdout}\n{r.stderr}")


def build_variant(name: str, defines: list) -> str:
    """A/B tuning build: the product library with extra -D defines, linked to
    lib/variants/libtttstate_<name>.so (loaded with TTT_LIB_PATH; never the default)."""
    vobj = os.path.join(OBJ, "variants", name)
    os.makedirs(vobj, exist_ok=True)
    out = os.path.join(LIB, "variants", f"libtttstate_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objs = []
    for src in PRODUCT_CU + PRODUCT_CPP:
        path = os.path.join(CSRC, src)
        obj = os.path.join(vobj, src.replace("/", "_") + ".o")
        dflags = [f"-D{d}" for d in defines]
        cmd = ([NVCC] + NVFLAGS if src.endswith(".cu") else ["g++"] + CXXFLAGS) + dflags + ["-c", path, "-o", obj]
        objs.append((cmd, obj))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        res = list(ex.map(lambda c: subprocess.run(c[0], capture_output=True, text=True), objs))
    for r in res:
        if r.returncode != 0:
            raise RuntimeError(r.stdout + r.stderr)
    _link([o for _, o in objs], out, True)
    return out


def build(force: bool = False, verbose: bool = False) -> dict:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    log: list = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        prod = list(ex.map(lambda s: _compile(s, force, log), PRODUCT_CU + PRODUCT_CPP))
        gen = list(ex.map(lambda s: _compile(s, force, log), GEN_CU))
    out_prod = os.path.join(LIB, "libtttstate.so")
    out_gen = os.path.join(LIB, "libttt_gen.so")
    _link(prod, out_prod, force)
    _link(gen, out_gen, force)
    if verbose:
        for src, text in log:
            print(f"== {src}\n{text}")
    return {"libtttstate": out_prod, "libttt_gen": out_gen, "log": log}


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":   # --variant NAME DEF=V ...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build(force="--force" in sys.argv, verbose=True)
