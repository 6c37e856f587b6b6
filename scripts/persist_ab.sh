timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for c in w8a covtype delicious realsim scaled; do for p in 0 1; do
  HB_NO_PERSIST=$p timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-budget-s 0.2 --ttt-epochs 0 --skip-e2e > gpurun_out/ps_${c}_$p.json 2>gpurun_out/ps_${c}_$p.err
  python -c "
import json; d=json.loads(open('gpurun_out/ps_${c}_$p.json').read().strip().splitlines()[-1])
k=d['kernels']
print('$c nopersist=$p', 'ms %.4f value %.4e'%(d['ms_per_step'], d['value']), d['roofline']['kernel'], d['roofline']['frac'])
print('   ', ' '.join('%s=%.1f'%(n,v['avg_us']) for n,v in k.items()))" || tail -3 gpurun_out/ps_${c}_$p.err
done; done
