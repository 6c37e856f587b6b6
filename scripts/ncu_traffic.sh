# One `ncu --set full` capture per (config, kernel), selected by the library's
# NVTX ranges (HB_NVTX=1, eager steps).  Raw pages land in gpurun_out/ncu_*.csv;
# scripts/ncu_summarize.py <round> turns them into profiles/<round>_ncu_kernels.json.
# KERNELS="config:kernel ..." overrides the list.
mkdir -p gpurun_out
run() {  # config kernel
  HB_NVTX=1 HB_NO_GRAPHS=1 timeout 900 ncu --set full --clock-control none --import-source on --nvtx \
      --nvtx-include "$2/" -c 2 -o gpurun_out/ncu_$1_$2 -f \
      python bench.py --config $1 --steps 2 --warmup 3 --skip-e2e --skip-cpu --no-prof --no-ttt \
      > gpurun_out/ncu_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
  ncu -i gpurun_out/ncu_$1_$2.ncu-rep --page raw --csv > gpurun_out/ncu_$1_$2.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$1_$2.ncu-rep --page details --csv > gpurun_out/ncu_$1_$2_details.csv 2>/dev/null
  if [ -n "$KEEP_REP" ]; then :; else rm -f gpurun_out/ncu_$1_$2.ncu-rep; fi
}
for ck in ${KERNELS:-scaled:gemm_dw_sgd_l1 scaled:gemm_dx_dsig_l2 scaled:gemm_fwd_sigmoid_l1 scaled:gemm_fwd_sigmoid_l2 scaled:gemm_fwd_logits_l3 scaled:gemm_dw_partial_l3 realsim:spmm_sigmoid_l0 realsim:sparse_dw_sgd_l0 realsim:gemm_fwd_sigmoid_l1 w8a:gemm_dx_dsig_l1}; do
  run ${ck%%:*} ${ck#*:}
done
ls -la gpurun_out/ncu_*.csv
