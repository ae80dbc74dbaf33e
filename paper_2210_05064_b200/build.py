"""Build the in-tree sm_100a library ``paper_2210_05064_b200/_lib/libver_b200.so``.

Explicit ``nvcc`` (no JIT cache): the .so is built here (CPU container,
nvcc cross-compiles) and travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libver_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3", "-I", str(ROOT / "include"), "-I", str(CSRC),
]
LDFLAGS = ARCH + ["-shared", "-L/usr/lib/x86_64-linux-gnu", "-lnccl"]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "ver_gpu.h"]


def _obj(src: Path) -> Path:
    return OUT_DIR / "obj" / (src.stem + ".o")


def _stale(target: Path, inputs: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    (OUT_DIR / "obj").mkdir(parents=True, exist_ok=True)
    deps = _deps()
    srcs = _sources()
    todo = [s for s in srcs if _stale(_obj(s), [s] + deps)]

    def compile_one(src: Path) -> tuple[Path, str]:
        cmd = [NVCC, *CFLAGS, "-c", str(src), "-o", str(_obj(src))]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        return src, r.stderr

    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        for src, err in ex.map(compile_one, todo):
            if verbose and err.strip():
                print(err, file=sys.stderr)
    objs = [_obj(s) for s in srcs]
    if todo or _stale(LIB, objs):
        cmd = [NVCC, *LDFLAGS, "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
