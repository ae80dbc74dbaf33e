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


def _nccl_dir() -> Path | None:
    """torch's bundled NCCL (nvidia-nccl wheel, 2.28): the library links against
    the same libnccl.so.2 torch loads, so one NCCL serves the whole process
    whichever of the two is imported first (the system 2.27 copy has the same
    soname and would shadow torch's if it were loaded first)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []) or []:
        d = Path(base) / "nccl"
        if (d / "lib" / "libnccl.so.2").exists() and (d / "include" / "nccl.h").exists():
            return d
    return None


NCCL = _nccl_dir()
_NCCL_INC = ["-I", str(NCCL / "include")] if NCCL else []
_NCCL_LIB = (["-Xlinker", str(NCCL / "lib" / "libnccl.so.2"), "-Xlinker", f"-rpath={NCCL / 'lib'}"] if NCCL
             else ["-L/usr/lib/x86_64-linux-gnu", "-lnccl"])
CFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3", *_NCCL_INC, "-I", str(ROOT / "include"), "-I", str(CSRC),
]
LDFLAGS = ARCH + ["-shared", *_NCCL_LIB]


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
