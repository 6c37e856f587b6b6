for cfg in "8 1" "8 2" "2 2" "8 8"; do set -- $cfg
echo "=== threads $1 parts $2"
for rep in 1 2; do
HB_MERGE_PARTS=$2 HB_HOST_MERGE_THREADS=$1 HB_XCHG_MERGE=host HB_DEBUG_XCHG=1 python scripts/xchg_timeline.py w8a 2>&1 | sed -n '/call 2/,$p' | grep -E "G. done|on host|end" | tr '\n' ' ' | sed 's/\[xchg\]//g; s/  */ /g'; echo
done
HB_MERGE_PARTS=$2 HB_HOST_MERGE_THREADS=$1 HB_XCHG_MERGE=host python scripts/e2e_probe3.py w8a 2>&1 | grep -E "replica_step"
done
