# every config's bench line (device value, e2e, roofline, CPU baselines, time-to-target) -> gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
for c in ${CONFIGS:-scaled w8a delicious realsim covtype}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); e=d['e2e']; r=d['roofline']; c=d.get('cpu_baseline') or {}; t=(d.get('time_to_target') or {}); print('$c ms/step %.4f value %.3e e2e %.3e cpu %.3e dom %s frac %.3f step_tensor %.3f ttt %s' % (d['ms_per_step'], d['value'], e['value'], c.get('value',0), r.get('kernel'), r.get('frac',0), r.get('step_tensor',{}).get('frac_of_peak',0), {k:v.get('speedup') for k,v in t.items() if isinstance(v,dict) and 'speedup' in v}))"
done
