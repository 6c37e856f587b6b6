timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in ${CONFIGS:-w8a covtype delicious realsim}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-budget-s 0.2 --ttt-epochs 0 --skip-e2e > gpurun_out/qb_$c.json 2>gpurun_out/qb_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/qb_$c.json').read().strip().splitlines()[-1])
k=d['kernels']
print('$c', 'ms %.4f value %.4e'%(d['ms_per_step'], d['value']), d['roofline']['kernel'], d['roofline']['frac'])
print('   ', ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in k.items()))" || tail -3 gpurun_out/qb_$c.err
done
