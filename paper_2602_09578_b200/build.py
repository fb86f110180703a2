"""Builds the native library ``_native/libflexmarl_b200.so`` in-tree.

All CUDA sources are compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's
source page maps back to the kernels.  nvcc cross-compiles without a GPU, so
this runs in the CPU container; the resulting .so travels to the GPU box with
the repo snapshot.  Usage: ``python -m paper_2602_09578_b200.build [-v]``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_native"
LIB = OUT_DIR / "libflexmarl_b200.so"
OBJ_DIR = ROOT / "build" / "obj"
# debug variant: device-side bounds checks (FM_DCHECK, fm_ptx.cuh) in place of
# compute-sanitizer, which the GPU pool does not offer; loaded with FLEXMARL_DEBUG_LIB=1
LIB_DEBUG = OUT_DIR / "libflexmarl_b200_debug.so"
OBJ_DIR_DEBUG = ROOT / "build" / "obj_debug"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> Path | None:
    """torch's bundled NCCL (2.28.x): linking and rpath-ing the same libnccl.so.2
    torch uses keeps one NCCL in the process whichever library loads first."""
    try:
        import nvidia.nccl  # type: ignore
        d = Path(list(nvidia.nccl.__path__)[0])
        if (d / "lib" / "libnccl.so.2").exists() and (d / "include" / "nccl.h").exists():
            return d
    except Exception:
        pass
    return None
CUDA_SOURCES = ["k_gemm_tc.cu", "k_band.cu", "k_path.cu", "k_rollout.cu", "k_store.cu", "fm_runtime.cu", "fm_swap.cu", "fm_gang.cu",
                "fm_publish.cu", "fm_dtable.cu"]
CXX_SOURCES = ["fm_host.cpp"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _flags() -> list[str]:
    return [
        "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
        f"-I{ROOT / 'include'}", f"-I{CSRC}",
        *([f"-I{nccl_dir() / 'include'}"] if nccl_dir() else []),
        "--expt-relaxed-constexpr",
    ]


def _compile(src: Path, obj: Path, verbose: bool, debug: bool = False) -> None:
    cmd = [nvcc(), *ARCH, *_flags(), *(["-DFM_DEBUG_CHECKS"] if debug else []), "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd.insert(1, "-Xptxas=-v") if verbose else None
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr, flush=True)


def _stale(outp: Path, deps: list[Path]) -> bool:
    if not outp.exists():
        return True
    t = outp.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, debug: bool = False) -> Path:
    obj_dir, lib = (OBJ_DIR_DEBUG, LIB_DEBUG) if debug else (OBJ_DIR, LIB)
    obj_dir.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").rglob("*.h"))
    jobs = []
    objs = []
    for name in CUDA_SOURCES + CXX_SOURCES:
        src = CSRC / name
        obj = obj_dir / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers]):
            jobs.append((src, obj))
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_compile, s, o, verbose, debug) for s, o in jobs]:
            f.result()
    if force or jobs or _stale(lib, objs):
        nd = nccl_dir()
        link = ([f"-L{nd / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nd / 'lib'}"] if nd
                else ["-lnccl"])
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), *link]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed\n{res.stdout}\n{res.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, debug="--debug" in sys.argv))
