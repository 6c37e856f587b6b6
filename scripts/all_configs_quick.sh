# GPU parity suite, then every config bench line (device value and e2e) -> gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for c in covtype w8a delicious realsim scaled; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); e=d['e2e']; print('$c ms/step %.4f value %.3e e2e %.3e seq %.3e' % (d['ms_per_step'], d['value'], e['value'], e['sequential']['value']))"
done
