# GPU parity tests of the opt-in persistent small-net step, then the covtype bench with it on and off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small_net.py -x -q -p no:cacheprovider > gpurun_out/small.log 2>&1; echo small_rc=$?; tail -30 gpurun_out/small.log
timeout 300 python bench.py --config covtype --skip-cpu --no-ttt > gpurun_out/cov_fused.json 2> gpurun_out/cov_fused.err; echo rc=$?
HB_SMALL_NET=0 timeout 300 python bench.py --config covtype --skip-cpu --no-ttt > gpurun_out/cov_layer.json 2> gpurun_out/cov_layer.err; echo rc=$?
python - <<'P'
import json
for n in ['cov_fused','cov_layer']:
    try:
        d=json.load(open(f'gpurun_out/{n}.json')); print(n, d['ms_per_step'], d['value'], d['e2e']['value'], d['gpu_launches'], list(d.get('kernels',{}).items())[:3])
    except Exception as e: print(n, 'ERR', e)
P
tail -5 gpurun_out/cov_fused.err
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_gpu.log
