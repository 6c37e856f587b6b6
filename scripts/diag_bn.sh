# precision vs tile width: per-layer parity diagnostics with capped GEMM tile widths
mkdir -p gpurun_out
for cfg in "" "HB_FWD_BN_MAX=128" "HB_FWD_BN_MAX=64" "HB_FWD_BN_MAX=64 HB_DX_BN_MAX=64 HB_DW_BN_MAX=64"; do
  for c in ${DIAG_CASES:-realsim delicious}; do
    echo "== [$cfg] $c"
    env $cfg timeout 600 python scripts/diag_layers.py $c 8192 ${DIAG_SEEDS:-1} 2>&1 | grep -E "csr-kernels|dense-l0" | grep -E " (A2|G1|G2|W1|W2):"
  done
done
