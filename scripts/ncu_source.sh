# source-level (SASS + CUDA line) stall profile of one kernel: $1 config, $2 NVTX kernel name
mkdir -p gpurun_out
HB_NVTX=1 HB_NO_GRAPHS=1 timeout 900 ncu --set full --clock-control none --import-source on --nvtx \
    --nvtx-include "$2/" -c 1 -o gpurun_out/src_$1_$2 -f \
    python bench.py --config $1 --steps 2 --warmup 3 --skip-e2e --no-prof --ttt-epochs 0 --cpu-budget-s 0.1 > /dev/null 2>&1
ncu -i gpurun_out/src_$1_$2.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1_$2.csv 2>&1
rm -f gpurun_out/src_$1_$2.ncu-rep
ls -la gpurun_out/src_$1_$2.csv
