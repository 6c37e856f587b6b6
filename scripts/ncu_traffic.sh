# One `ncu --set full` capture per (config, kernel): the dominant kernel of each
# bench config plus the sparse first-layer kernels, selected by the library's
# NVTX ranges (HB_NVTX=1, eager steps).  Raw pages land in gpurun_out/ncu_*.csv.
mkdir -p gpurun_out
run() {  # config kernel
  HB_NVTX=1 HB_NO_GRAPHS=1 timeout 900 ncu --set full --clock-control none --import-source on --nvtx \
      --nvtx-include "$2/" -c 3 -o gpurun_out/ncu_$1_$2 -f \
      python bench.py --config $1 --steps 2 --warmup 3 --skip-e2e --no-prof --ttt-epochs 0 --cpu-budget-s 0.1 \
      > gpurun_out/ncu_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
  ncu -i gpurun_out/ncu_$1_$2.ncu-rep --page raw --csv > gpurun_out/ncu_$1_$2.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$1_$2.ncu-rep --page details --csv > gpurun_out/ncu_$1_$2_details.csv 2>/dev/null
  rm -f gpurun_out/ncu_$1_$2.ncu-rep
}
run w8a gemm_dx_dsig_l2
run w8a gemm_dx_dsig_l1
run w8a gemm_dw_partial_l1
run w8a gemm_fwd_sigmoid_l1
run w8a gemm_dw_partial_l2
run w8a head_small_l3
run covtype gemm_fwd_sigmoid_l1
run covtype gemm_dx_dsig_l1
run delicious gemm_dx_dsig_l2
run delicious gemm_dw_partial_l2
run realsim sparse_dw_sgd_l0
run realsim spmm_sigmoid_l0
run scaled gemm_dw_sgd_l1
run scaled gemm_dx_dsig_l2
ls -la gpurun_out/ncu_*.csv
