"""Builds libds2ctc.so in-tree (sm_100a only) with nvcc.

    python -m paper_1512_02595_b200.build [--force]

The library is a plain C-ABI shared object (include/ds2ctc.h); the CUDA
runtime is linked statically so the .so carries no torch or libcudart
dependency and travels to the GPU box as-is.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libds2ctc.so")
BUILD = os.path.join(PKG, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["ctc_pair.cu", "ctc_pair_k8.cu", "ctc_dense.cu", "ctc_viterbi.cu", "ctc_lattice.cu", "ctc_reduce.cu",
              "fc_backward.cu"]
# Per-source extra flags. ctc_pair_k8.cu: ptxas 12.9 -O3 segfaults on the
# K = 8 pair kernel at its 168-register budget; -O1 builds it without spills.
CU_FLAGS = {"ctc_pair_k8.cu": ["-Xptxas", "-O1"]}
CPP_SOURCES = ["ctc_api.cpp", "scheduler.cpp"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _content_hash(deps, flags) -> str:
    """sha256 over every source's bytes, the build flags and the compiler version:
    a prebuilt library is reused only if it was built from exactly these inputs
    (modification times are not trusted: a snapshot copy can reorder them)."""
    h = hashlib.sha256()
    for d in sorted(deps):
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(flags).encode())
    try:
        h.update(subprocess.run([nvcc(), "--version"], capture_output=True, text=True).stdout.encode())
    except Exception:
        pass
    return h.hexdigest()


def _up_to_date(lib: str, digest: str) -> bool:
    try:
        with open(lib + ".sha256") as f:
            return os.path.exists(lib) and f.read().strip() == digest
    except OSError:
        return False


def check_no_stack(src: str, ptxas_log: str) -> None:
    """Refuses kernels that need a local-memory stack frame (register spills).

    ptxas 12.9 for sm_100a was seen to reuse R1 -- the stack pointer -- as a
    general register in the spilling k_pair<8> instantiation, so its STL/LDL
    hit wild local addresses (an illegal-address fault only for some label
    lengths). The kernels are written to fit in registers; a build that spills
    fails here instead of shipping."""
    cur = None
    for line in ptxas_log.splitlines():
        if "Function properties for" in line:
            cur = line.split("Function properties for")[-1].strip()
        elif cur and "bytes stack frame" in line:
            frame = int(line.strip().split()[0])
            if frame and "watchdog" not in cur:
                raise RuntimeError(f"{src}: {cur} needs a {frame}-byte stack frame (register spill); "
                                   "refusing the build (see build.check_no_stack)")
            cur = None


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, build_dir: str = BUILD) -> str:
    """Builds the library. `defines` (debug experiments only, e.g. ("DS2CTC_EXP_NOOCC",))
    go to a separate `lib` / `build_dir`; the product library is built without any."""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if os.path.isfile(os.path.join(CSRC, f))]
    deps += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith((".h", ".hpp"))] + [__file__]
    digest = _content_hash(deps, [*ARCH, *defines])
    if not force and _up_to_date(lib, digest):
        return lib
    LIB_ = lib
    BUILD_ = build_dir
    os.makedirs(BUILD_, exist_ok=True)
    cc = nvcc()
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", f"-I{INCLUDE}", f"-I{CSRC}",
              *[f"-D{d}" for d in defines]]
    objs = []
    for src in CU_SOURCES:
        obj = os.path.join(BUILD_, src + ".o")
        cmd = [cc, *ARCH, "-lineinfo", "-Xptxas", "-v", *CU_FLAGS.get(src, []), *common, "-c", os.path.join(CSRC, src),
               "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stderr}")
        with open(os.path.join(BUILD_, src + ".ptxas.txt"), "w") as f:
            f.write(res.stderr)
        check_no_stack(src, res.stderr)
        if verbose:
            print(res.stderr)
        objs.append(obj)
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(cc)), "include")
    for src in CPP_SOURCES:
        obj = os.path.join(BUILD_, src + ".o")
        cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", f"-I{INCLUDE}",
               f"-I{CSRC}", f"-I{cuda_inc}", *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB_ + ".tmp"
    subprocess.run([cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread", "-ldl", "-lrt"],
                   check=True)
    os.replace(tmp, LIB_)
    with open(LIB_ + ".sha256", "w") as f:
        f.write(digest + "\n")
    return LIB_


def build_variant(name: str, defines) -> str:
    """Debug-experiment library build/variants/libds2ctc_<name>.so (bench.py picks
    it up through DS2CTC_LIB); never used by the product path."""
    out = os.path.join(ROOT, "build", "variants")
    return build(force=True, defines=defines, lib=os.path.join(out, f"libds2ctc_{name}.so"),
                 build_dir=os.path.join(out, name))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
