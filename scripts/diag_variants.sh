# per-layer parity diagnostics under library variants (precision A/B)
mkdir -p gpurun_out
for v in ${VARIANTS:-default}; do
  lib=paper_2004_08771_b200/libhogbatch_b200.so; [ "$v" != default ] && lib=build_variants/$v.so
  for c in ${DIAG_CASES:-realsim}; do
    echo "== $v $c"
    HOGBATCH_B200_LIB=$lib timeout 600 python scripts/diag_layers.py $c ${DIAG_B:-8192} ${DIAG_SEEDS:-8199 1 2}
  done
done
