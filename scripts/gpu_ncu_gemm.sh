# one full ncu capture of the forward GEMM (3xTF32) + the launch list
python -m paper_2004_08771_b200.build >/dev/null
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel -s 13 -c 2 -o gpurun_out/prof_gemm2 -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 0.1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches2.csv \
    python bench.py --steps 3 --warmup 3 --skip-e2e --cpu-budget-s 0.1 > /dev/null 2>&1
ls -la gpurun_out/
