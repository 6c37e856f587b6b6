# launch list (cold-cache, serialised) + one full capture of the top GEMM and the sparse kernels
set -x
mkdir -p gpurun_out
python -m paper_2004_08771_b200.build >/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --cpu-budget-s 1 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 10 -c 3 -o gpurun_out/prof_gemm -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sparse_dw|spmm|head_small|reduce_sgd" -s 4 -c 4 -o gpurun_out/prof_sparse -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 1 > /dev/null 2>&1
ls -la gpurun_out
