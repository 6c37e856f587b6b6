for m in host dma; do
echo "=== $m"
HB_XCHG_MERGE=$m HB_DEBUG_XCHG=1 python scripts/xchg_timeline.py w8a 2>&1 | sed -n '/call 2/,$p'
done
