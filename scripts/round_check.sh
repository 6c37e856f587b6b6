# full check: smoke, GPU parity tests, default bench, every config, launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
cat gpurun_out/bench_default.json
for c in covtype delicious realsim scaled; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget-s 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
cat gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --cpu-budget-s 0.1 --ttt-epochs 0 > gpurun_out/bench_under_ncu.log 2>&1
echo ncu_rc=$?
