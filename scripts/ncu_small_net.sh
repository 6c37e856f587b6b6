# one ncu --set full capture of the persistent small-net step (covtype config)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:small_net -s 2 -c 1 -o gpurun_out/small_net -f \
  python bench.py --config covtype --steps 3 --warmup 3 --skip-e2e --skip-cpu --no-ttt > gpurun_out/ncu_small.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_small.log
