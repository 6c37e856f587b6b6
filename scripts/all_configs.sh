# every BASELINE.json config through bench.py (device value, e2e, roofline), one JSON line each
mkdir -p gpurun_out
for c in covtype w8a delicious realsim scaled; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget-s 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 600 gpurun_out/bench_$c.err
done
