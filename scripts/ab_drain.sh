# Accumulator drain policy sweep: per-layer precision and step times (HB_DRAIN_KB_CRIT: precision-critical
# GEMMs, HB_DRAIN_KB: all others; 0 = rotating accumulators)
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_drain.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_drain.log
fi
for cfg in ${DRAIN_CFGS:-"HB_DRAIN_KB_CRIT=0" "HB_DRAIN_KB_CRIT=1" "HB_DRAIN_KB_CRIT=2" "HB_DRAIN_KB_CRIT=3" "HB_DRAIN_KB_CRIT=1 HB_DRAIN_KB=4"}; do
  for c in realsim delicious scaled; do
    echo "== [$cfg] $c"
    env $cfg timeout 600 python scripts/diag_layers.py $c 8192 ${DIAG_SEEDS:-1} 2>&1 | grep -E "(csr-kernels|dense-l0) (G2|G3|W1|W2|W3):" | sed -E 's/ at \(np.int64\(([0-9]+)\), np.int64\(([0-9]+)\)\)//; s/\(gpu[^)]*\)//' | cut -c1-120 | sort -u
  done
  for c in w8a delicious realsim scaled covtype; do
    env $cfg timeout 300 python bench.py --config $c --steps 20 --warmup 5 --skip-e2e --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$cfg] $c ms/step %.4f step_tensor %.3f' % (d['ms_per_step'], d['roofline'].get('step_tensor',{}).get('frac_of_peak',0)))"
  done
done
