"""Build the in-tree CUDA engine: ``paper_2311_02840_b200/_lib/libsaturn_b200.so``.

Plain nvcc, sm_100a only, static cudart (the .so loads through ctypes without
any CUDA runtime on the library path).  The walk kernel is specialised for
every node size 1..32, so its instantiations are split over several
translation units compiled in parallel.  The built file is git-ignored but
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HDR = os.path.join(ROOT, "include", "saturn_engine.h")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
OUT = os.path.join(OUT_DIR, "libsaturn_b200.so")
# debug variant: device-side bounds checks on every shared-memory region index (SAT_ASSERT)
DEBUG_OBJ_DIR = os.path.join(OUT_DIR, "obj_debug")
DEBUG_OUT = os.path.join(OUT_DIR, "libsaturn_b200_debug.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "128"]
TREE_RANGES = [(1, 6), (7, 10), (11, 14), (15, 18), (19, 22), (23, 26), (27, 29), (30, 32)]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [HDR]


def up_to_date(out_path: str = OUT) -> bool:
    if not os.path.exists(out_path):
        return False
    t = os.path.getmtime(out_path)
    return all(os.path.getmtime(f) <= t for f in sources() + [__file__])


def _obj_fresh(src: str, obj: str) -> bool:
    """An object is reused when it is newer than its own .cu, every header and this file."""
    if not os.path.exists(obj):
        return False
    deps = [src, HDR, __file__] + glob.glob(os.path.join(CSRC, "*.cuh"))
    t = os.path.getmtime(obj)
    return all(os.path.getmtime(f) <= t for f in deps)


def units(obj_dir: str = OBJ_DIR) -> list:
    """(source, extra defines, object) for every translation unit."""
    OBJ_DIR = obj_dir  # noqa: N806 (local rebinding keeps the table below readable)
    out = [(os.path.join(CSRC, "sat_engine.cu"), [], os.path.join(OBJ_DIR, "sat_engine.o")),
           (os.path.join(CSRC, "sat_dp.cu"), [], os.path.join(OBJ_DIR, "sat_dp.o"))]
    for t in ("int32_t", "double"):
        for s in ("SAT_SRC_INDEX", "SAT_SRC_SUBSTREAM", "SAT_SRC_SEED"):
            ls = ["-DSAT_LS_INSTANTIATE"] if t == "int32_t" and s != "SAT_SRC_INDEX" else []
            out.append((os.path.join(CSRC, "sat_cand.cu"), [f"-DSAT_CAND_T={t}", f"-DSAT_CAND_SRC={s}", *ls],
                        os.path.join(OBJ_DIR, f"sat_cand_{t}_{s.split('_')[-1].lower()}.o")))
    for lo, hi in TREE_RANGES:
        out.append((os.path.join(CSRC, "sat_tree_g.cu"), [f"-DSAT_G_LO={lo}", f"-DSAT_G_HI={hi}"],
                    os.path.join(OBJ_DIR, f"sat_tree_g{lo}_{hi}.o")))
    return out


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    out_path, obj_dir = (DEBUG_OUT, DEBUG_OBJ_DIR) if debug else (OUT, OBJ_DIR)
    extra = ["-DSAT_DEBUG_BOUNDS"] if debug else []
    if not force and up_to_date(out_path):
        return out_path
    os.makedirs(obj_dir, exist_ok=True)
    cc = nvcc()
    procs = []
    for src, defs, obj in units(obj_dir):
        if not force and _obj_fresh(src, obj):
            continue
        cmd = [cc, *NVCC_FLAGS, *extra, *defs, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    tmp = out_path + ".tmp"
    link = [cc, *ARCH, "-shared", "-o", tmp, *[obj for _, _, obj in units(obj_dir)]]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(tmp, out_path)
    return out_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
