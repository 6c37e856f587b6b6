# A/B of the GEMM accumulator drain: parity suite, per-layer precision, step times per config
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_drain.log 2>&1; echo "pytest(drain) rc=$?"; tail -15 gpurun_out/pytest_drain.log
for v in default nodrain; do
  lib=paper_2004_08771_b200/libhogbatch_b200.so; [ "$v" != default ] && lib=build_variants/$v.so
  for c in realsim delicious scaled; do
    echo "== $v $c"
    HOGBATCH_B200_LIB=$lib timeout 600 python scripts/diag_layers.py $c 8192 1 2>&1 | grep -E " (A2|A3|G1|G2|G3|W1|W2|W3):" | grep -v dense-l0 ; true
    HOGBATCH_B200_LIB=$lib timeout 600 python scripts/diag_layers.py $c 8192 1 2>&1 | grep -E "dense-l0 (A2|A3|G2|G3|W2|W3):" | head -6
  done
  for c in w8a delicious realsim scaled covtype; do
    HOGBATCH_B200_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --skip-e2e --skip-cpu --no-ttt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] $c ms/step %.4f step_tensor %.3f' % (d['ms_per_step'], d['roofline'].get('step_tensor',{}).get('frac_of_peak',0)))"
  done
done
