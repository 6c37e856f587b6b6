echo "=== tf32 default lib"; python bench.py --steps 10 --warmup 3 --skip-e2e --cpu-budget-s 0.5 --precision tf32 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in k.items() if 'gemm' in n))"
echo "=== nostore"; HOGBATCH_B200_LIB=$PWD/build_variants/nostore.so python bench.py --steps 10 --warmup 3 --skip-e2e --cpu-budget-s 0.5 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in k.items() if 'gemm' in n))"
