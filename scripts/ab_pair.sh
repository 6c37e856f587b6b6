timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
HOGBATCH_B200_LIB=$PWD/build_variants/trace.so timeout 60 python scripts/trace_gemm.py > /tmp/o1 2>&1; head -8 /tmp/o1
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-budget-s 0.5 --skip-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('ms/step %.3f value %.3e'%(d['ms_per_step'], d['value']))
print('   ', ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['avg_us'])))"
