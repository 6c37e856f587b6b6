mkdir -p gpurun_out
for ml in "" "all"; do
for c in scaled w8a realsim; do
  HB_MIRROR_LANE=$ml timeout 600 python bench.py --config $c --steps 20 --warmup 5 --skip-cpu --no-ttt --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('[mirror_lane=$ml] $c e2e %.3e h2d %d d2h %d' % (e['value'], e['h2d_bytes_per_step'], e['d2h_bytes_per_step']))"
done
done
timeout 600 python bench.py --config w8a --steps 5 --warmup 3 --skip-cpu --skip-e2e --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['time_to_target']; print({k:(v.get('gpu_steps'), v.get('speedup'), v.get('target_loss')) for k,v in t.items() if isinstance(v,dict)})"
