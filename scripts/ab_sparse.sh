# CSR gather kernel variants (register cap / gathers in flight): real-sim step and kernel times
for v in ${VARIANTS:-default sp_m4 sp_p4m5 sp_p4m6 sp_p4m8 sp_p2m8}; do
  lib=paper_2004_08771_b200/libhogbatch_b200.so; [ "$v" != default ] && lib=build_variants/$v.so
  for rep in 1; do
  HOGBATCH_B200_LIB=$lib timeout 300 python bench.py --config realsim --steps 20 --warmup 5 --skip-e2e --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('[$v] realsim ms/step %.4f spmm %.1f us sparse_dw %.1f us' % (d['ms_per_step'], k.get('spmm_sigmoid_l0',{}).get('avg_us',0), k.get('sparse_dw_sgd_l0',{}).get('avg_us',0)))"
  done
done
