for m in host dma; do
  HB_XCHG_MERGE=$m timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or stale or execute" 2>&1 | grep -E "Error|error|passed|failed" | head -5
done
for m in host dma; do
HB_XCHG_MERGE=$m HB_DEBUG_XCHG=1 python scripts/xchg_timeline.py w8a 2>&1 | tail -36
done
for m in host dma; do for c in w8a covtype delicious realsim scaled; do
  echo "== $m $c"; HB_XCHG_MERGE=$m python scripts/e2e_probe3.py $c 2>&1 | grep -E "replica_step|step_host \(|Error"
done; done
