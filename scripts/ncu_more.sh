source <(sed -n '/^run() {/,/^}/p' scripts/ncu_traffic.sh)
mkdir -p gpurun_out
run scaled gemm_dx_dsig_l2
