"""Build a tuning variant of libstam_cuda.so with extra -D flags into
paper_1802_10574_b200/_lib/variants/<name>/ (load it with STAM_CUDA_LIB).

    python tools/build_variant.py w16r1 -DSPADD_WARPS=16 -DSPADD_RPW=1
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1802_10574_b200 import _build as B  # noqa: E402


def main(name, *defs):
    out_dir = B.LIB / "variants" / name
    obj_dir = B.OBJ / "variants" / name
    out_dir.mkdir(parents=True, exist_ok=True)
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = B._nvcc()
    objs = []
    for src in B.CUDA_SOURCES:
        s = B.CSRC / src
        o = obj_dir / (s.stem + ".o")
        lang = ["-x", "cu"] if s.suffix == ".cpp" else []
        B._run([nvcc, *B.ARCH, *B.NVCC_FLAGS, *defs, *lang, "-c", str(s), "-o", str(o)], False)
        objs.append(o)
    out = out_dir / "libstam_cuda.so"
    B._run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs),
            "-Xlinker", "-Bsymbolic"], False)
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
