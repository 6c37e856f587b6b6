# quick GPU check: parity tests + bench summary (optionally with extra env / args)
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for env in "" "HB_NO_GRAPHS=1"; do
env $env python bench.py --steps 20 --warmup 5 --cpu-budget-s 0.5 ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('[$env] ms/step %.3f value %.3e e2e %.3e launches %d'%(d['ms_per_step'], d['value'], d['e2e']['value'] if d['e2e'] else 0, d['gpu_launches']))
print('   ', ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['avg_us'])))"
done
