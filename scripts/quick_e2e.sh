# GPU: fused replica step parity + e2e of every config
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or stale or execute" > gpurun_out/pytest_fused.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_fused.log
for c in ${CONFIGS:-w8a covtype delicious realsim scaled}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget-s 0.5 --ttt-epochs 0 --no-prof > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_$c.json').read().strip().splitlines()[-1])
print('$c', 'ms %.3f value %.3e e2e %.3e'%(d['ms_per_step'], d['value'], d['e2e']['value']))" || tail -5 gpurun_out/e2e_$c.err
done
