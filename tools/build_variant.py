"""Build a tuning variant of libstam_cuda.so with extra -D flags into
paper_1802_10574_b200/_lib/variants/<name>/ (load it with STAM_CUDA_LIB).

    python tools/build_variant.py w16r1 -DSPADD_WARPS=16 -DSPADD_RPW=1
    python tools/build_variant.py m4 --only=mttkrp.cu -DSPM_MINB=4   # other objects from the base build
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1802_10574_b200 import _build as B  # noqa: E402


def main(name, *defs):
    only = [d.split("=", 1)[1] for d in defs if d.startswith("--only=")]
    defs = [d for d in defs if not d.startswith("--only=")]
    out_dir = B.LIB / "variants" / name
    obj_dir = B.OBJ / "variants" / name
    out_dir.mkdir(parents=True, exist_ok=True)
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = B._nvcc()
    objs = []
    for src in B.CUDA_SOURCES:
        s = B.CSRC / src
        o = obj_dir / (s.stem + ".o")
        if only and src not in only:
            objs.append(B.OBJ / (s.stem + ".o"))  # unchanged: the base build's object
            continue
        lang = ["-x", "cu"] if s.suffix == ".cpp" else []
        B._run([nvcc, *B.ARCH, *B.NVCC_FLAGS, *defs, *lang, "-c", str(s), "-o", str(o)], False)
        objs.append(o)
    out = out_dir / "libstam_cuda.so"
    B._run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs),
            "-Xlinker", "-Bsymbolic"], False)
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
