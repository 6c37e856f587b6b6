python -m paper_2004_08771_b200.build >/dev/null
HB_SPARSE_SMEM=1 ncu --set full --clock-control none --import-source on -k regex:"smem_kernel" -s 2 -c 2 -o gpurun_out/prof_sparse3 -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 0.1 --ttt-epochs 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sparse_dw_kernel|spmm_sigmoid_kernel" -s 2 -c 2 -o gpurun_out/prof_sparse4 -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 0.1 --ttt-epochs 0 > /dev/null 2>&1
ls -la gpurun_out/prof_sparse*.ncu-rep
