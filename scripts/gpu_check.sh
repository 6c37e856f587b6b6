# GPU check: smoke, GPU parity tests, the default (headline) bench line, the reference arm
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
cat gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
fi
if [ -n "$REF" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
cat gpurun_out/bench_ref.json
fi
