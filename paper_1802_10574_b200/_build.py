"""Build recipes for the in-tree native libraries.

* ``_lib/libstam_cuda.so`` — the sm_100a kernels + C ABI (``include/stam_cuda.h``),
  compiled with ``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo``,
  static cudart so it does not depend on the runtime torch happens to load.
* ``_lib/libstam_cxx.so`` — the C++ API (``include/stam/*.h``: the reference's
  storage/format/workspace/error surface plus ``kernels.h``) over the C ABI.
* ``_lib/libstamgen.so`` — seeded synthetic input generators.
* ``oracle/liboracle.so`` and ``oracle/_ref/libstamref.so`` — the parity
  checkers (test infrastructure; ``oracle/Makefile``).

Everything is built in-tree so the ``.so`` files travel with the repo snapshot
to the GPU box.  nvcc cross-compiles for sm_100a without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib"
INCLUDE = ROOT / "include"
OBJ = ROOT / "build" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", str(INCLUDE), "-I", str(CSRC)]

CUDA_SOURCES = ["runtime.cpp", "index.cu", "spadd.cu", "spgemm.cu", "mttkrp.cu", "coiter.cu"]
CXX_SOURCES = ["host/error.cpp", "host/format.cpp", "host/storage.cpp", "host/workspace.cpp",
               "host/kernels.cpp", "host/io.cpp", "host/execute.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _cxx() -> str:
    # the image's $CXX wrapper works; fall back to the system compiler
    for cand in ("/usr/bin/g++", os.environ.get("CXX"), shutil.which("g++")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("g++ not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print("+", " ".join(cmd), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"build command failed: {' '.join(cmd[:3])} ...")


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(INCLUDE.rglob("*.h"))


def build_cuda(verbose: bool = False, force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    OBJ.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    hdrs = _headers()
    jobs = []
    for src in CUDA_SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            lang = ["-x", "cu"] if s.suffix == ".cpp" else []
            jobs.append([nvcc, *ARCH, *NVCC_FLAGS, *lang, "-c", str(s), "-o", str(o)])
    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, j, verbose) for j in jobs]:
            f.result()
    out = LIB / "libstam_cuda.so"
    if force or _stale(out, objs):
        _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs),
              "-Xlinker", "-Bsymbolic"], verbose)
    return out


def build_cxx(verbose: bool = False, force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    srcs = [CSRC / s for s in CXX_SOURCES]
    out = LIB / "libstam_cxx.so"
    cuda_so = LIB / "libstam_cuda.so"
    if force or _stale(out, srcs + _headers() + [cuda_so]):
        _run([_cxx(), "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
              "-I", str(INCLUDE), "-o", str(out), *map(str, srcs),
              "-L", str(LIB), "-lstam_cuda", "-Wl,-rpath,$ORIGIN"], verbose)
    return out


def build_gen(verbose: bool = False, force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    src = PKG / "gen" / "stam_gen.cpp"
    out = LIB / "libstamgen.so"
    if force or _stale(out, [src]):
        _run([_cxx(), "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-Wall",
              "-fvisibility=hidden", "-o", str(out), str(src)], verbose)
    return out


def build_oracle(verbose: bool = False, force: bool = False) -> None:
    """Builds oracle/liboracle.so and, when /root/reference exists, oracle/_ref."""
    args = ["make", "-s", "-C", str(ROOT / "oracle")]
    if force:
        args.append("-B")
    args += [f"CC={shutil.which('gcc') or 'gcc'}", f"CXX={_cxx()}"]
    _run(args, verbose)


def build_all(verbose: bool = False, force: bool = False) -> None:
    build_cuda(verbose, force)
    build_gen(verbose, force)
    if (CSRC / "host" / "kernels.cpp").exists():
        build_cxx(verbose, force)
    build_oracle(verbose, force)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv, force="-f" in sys.argv)
