nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)"
for t in 1 4 8; do for sp in 0 20000; do
echo "=== threads $t spin $sp"
HB_POOL_SPIN=$sp HB_HOST_MERGE_THREADS=$t HB_XCHG_MERGE=host HB_DEBUG_XCHG=1 python scripts/xchg_timeline.py w8a 2>&1 | sed -n '/call 2/,$p' | grep -E "G. done|on host|end"
HB_POOL_SPIN=$sp HB_HOST_MERGE_THREADS=$t HB_XCHG_MERGE=host python scripts/e2e_probe3.py w8a 2>&1 | grep -E "replica_step"
done; done
