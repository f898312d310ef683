for v in base "$@"; do
  if [ "$v" = base ]; then unset STAM_CUDA_LIB; else export STAM_CUDA_LIB=paper_1802_10574_b200/_lib/variants/$v/libstam_cuda.so; fi
  echo "== $v"; timeout 600 python tools/suite_spadd_k.py 2>&1 | grep workspace | tr '\n' ' '; echo
done
