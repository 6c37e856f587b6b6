mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "fused or device_lane or concurrent or pipelined or merge_grads" > gpurun_out/pytest_mirror.log 2>&1; echo "pytest(mirror) rc=$?"; tail -5 gpurun_out/pytest_mirror.log
for c in scaled w8a delicious realsim covtype; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --skip-cpu --no-ttt > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); e=d['e2e']; print('$c ms/step %.4f value %.3e e2e %.3e h2d %d d2h %d' % (d['ms_per_step'], d['value'], e['value'], e['h2d_bytes_per_step'], e['d2h_bytes_per_step']))"
done
HB_NO_MIRROR=1 timeout 600 python bench.py --config scaled --steps 20 --warmup 5 --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('[no mirror] scaled e2e %.3e h2d %d' % (e['value'], e['h2d_bytes_per_step']))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_scaled.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --skip-cpu --no-ttt > gpurun_out/bench_under_ncu.log 2>&1; echo "launch list rc=$?"
