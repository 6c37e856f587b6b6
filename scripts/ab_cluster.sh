timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
HOGBATCH_B200_LIB=$PWD/build_variants/trace.so python scripts/trace_gemm.py > /tmp/o1 2>&1; head -8 /tmp/o1
for cm in 1 2 4; do
HB_CLUSTER_M=$cm python bench.py --steps 20 --warmup 5 --cpu-budget-s 0.5 --skip-e2e ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('[cm=$cm] ms/step %.3f value %.3e'%(d['ms_per_step'], d['value']))
print('   ', ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['avg_us'])))"
done
