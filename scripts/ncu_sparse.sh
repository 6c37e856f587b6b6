python -m paper_2004_08771_b200.build >/dev/null
ncu --set full --clock-control none --import-source on -k regex:"smem_kernel" -s 2 -c 2 -o gpurun_out/prof_sparse2 -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 0.1 > /dev/null 2>&1
ls -la gpurun_out/prof_sparse2.ncu-rep
