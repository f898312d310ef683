#!/bin/bash
# usage: tools/sweep_variants.sh CONFIG VARIANT... (on the GPU box): kernel ms per variant
C=$1; shift
for v in base "$@"; do
  if [ "$v" = base ]; then unset STAM_CUDA_LIB; else export STAM_CUDA_LIB=paper_1802_10574_b200/_lib/variants/$v/libstam_cuda.so; fi
  r=$(timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['kernel_ms'],4), round(d['roofline']['frac'],3), 'step', round(d['ms_per_step'],4))")
  echo "$v $r"
done
