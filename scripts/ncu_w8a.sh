mkdir -p gpurun_out
# full capture of one step's GEMMs (w8a): fwd l0..l2, dX l2, dW l2, dX l1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 24 -c 6 -o gpurun_out/w8a_gemms -f \
    python bench.py --steps 2 --warmup 3 --skip-e2e --cpu-budget-s 0.1 --ttt-epochs 0 --no-prof > gpurun_out/ncu_w8a.log 2>&1
echo rc=$?
ncu -i gpurun_out/w8a_gemms.ncu-rep --page raw --csv > gpurun_out/w8a_gemms_raw.csv
ls -la gpurun_out/w8a_gemms*
