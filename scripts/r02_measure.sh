# round-2 measurements: ncu captures, launch list of the default bench, L2-gather ceiling, A/B switches
mkdir -p gpurun_out
bash scripts/ncu_traffic.sh > gpurun_out/ncu_traffic.log 2>&1; tail -12 gpurun_out/ncu_traffic.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_scaled.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --skip-cpu --no-ttt > gpurun_out/bench_under_ncu.log 2>&1; echo "launch list rc=$?"
python - <<'PY'
import paper_2004_08771_b200 as hb, ctypes as C
lib = hb.load_library()
for rows, cols in ((20958, 1024), (300, 512), (2_000_000, 1024)):
    for u in (1, 2, 4):
        v = C.c_double(0)
        rc = lib.hb_probe_l2_gather(0, rows, cols, 64, u, C.byref(v))
        print(f"l2_gather rows={rows} cols={cols} unroll={u}: {v.value:.1f} GB/s rc={rc}")
PY
for env in "" "HB_NO_L2_WINDOW=1"; do
  env $env timeout 300 python bench.py --config realsim --steps 20 --warmup 5 --skip-e2e --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('[$env] realsim ms/step %.4f spmm %.1f us sparse_dw %.1f us' % (d['ms_per_step'], k.get('spmm_sigmoid_l0',{}).get('avg_us',0), k.get('sparse_dw_sgd_l0',{}).get('avg_us',0)))"
done
for env in "" "HB_NO_CONC_BWD=1"; do
  for c in scaled delicious w8a; do
  env $env timeout 300 python bench.py --config $c --steps 20 --warmup 5 --skip-e2e --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$env] $c ms/step %.4f dominant %s frac %.3f step_tensor %.3f' % (d['ms_per_step'], r.get('kernel'), r.get('frac',0), r.get('step_tensor',{}).get('frac_of_peak',0)))"
  done
done
