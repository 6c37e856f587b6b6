# ncu launch list (serialized per-kernel durations) of the covtype bench
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_covtype.csv \
    python bench.py --config covtype --steps 3 --warmup 3 --skip-e2e --skip-cpu --no-ttt > gpurun_out/bench_cov_ncu.log 2>&1
echo ncu_rc=$?
