# full round check on one B200: smoke, GPU parity suite, every config's bench line, the reference arm,
# the launch list of the default bench (ncu), the sanitizer and knob-matrix passes
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
REF=1 bash scripts/gpu_check.sh
bash scripts/all_configs.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_scaled.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --skip-cpu --no-ttt > gpurun_out/bench_under_ncu.log 2>&1
echo ncu_rc=$?
# (compute-sanitizer is closed on this pool: bash scripts/sanitize.sh)
bash scripts/knob_matrix.sh
