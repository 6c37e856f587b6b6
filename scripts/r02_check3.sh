mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "fused or device_lane or concurrent or pipelined or merge_grads or pcie" > gpurun_out/pytest_mirror.log 2>&1; echo "pytest(mirror) rc=$?"; tail -5 gpurun_out/pytest_mirror.log
for ml in 1 0; do
for c in scaled w8a delicious realsim covtype; do
  HB_MIRROR_LANE=$ml timeout 600 python bench.py --config $c --steps 20 --warmup 5 --skip-cpu --no-ttt --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('[mirror_lane=$ml] $c ms/step %.4f value %.3e e2e %.3e h2d %d d2h %d' % (d['ms_per_step'], d['value'], e['value'], e['h2d_bytes_per_step'], e['d2h_bytes_per_step']))"
done
done
