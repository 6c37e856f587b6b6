timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in w8a covtype delicious realsim scaled; do for p in 0 1; do
  HB_NO_PDL=$p timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-budget-s 0.2 --ttt-epochs 0 > gpurun_out/pdl_$c_$p.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pdl_$c_$p.json').read().strip().splitlines()[-1])
print('$c nopdl=$p', 'ms %.4f value %.4e e2e %.3e'%(d['ms_per_step'], d['value'], d['e2e']['value']), d['roofline']['kernel'], d['roofline']['frac'])"
done; done
