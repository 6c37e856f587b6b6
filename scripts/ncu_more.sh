source <(sed -n '/^run() {/,/^}/p' scripts/ncu_traffic.sh)
mkdir -p gpurun_out
run w8a gemm_dx_dsig_l1
run w8a gemm_dw_partial_l1
run covtype gemm_dx_dsig_l1
run delicious gemm_dw_partial_l2
