# A/B the experimental library builds in build_variants/ against the default one
for v in paper_2004_08771_b200/libhogbatch_b200.so build_variants/*.so; do
  echo "=== $v"
  HOGBATCH_B200_LIB=$PWD/$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
  HOGBATCH_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --skip-e2e --cpu-budget-s 0.5 ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.1f'%(n.replace('gemm_','').replace('_sigmoid','').replace('_dsig','').replace('_partial',''),v['avg_us']) for n,v in k.items()))"
done
