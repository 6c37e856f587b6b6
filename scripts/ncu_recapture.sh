source <(sed -n '/^run() {/,/^}/p' scripts/ncu_traffic.sh)
mkdir -p gpurun_out
run realsim sparse_dw_sgd_l0
run covtype gemm_fwd_sigmoid_l1
run realsim spmm_sigmoid_l0
