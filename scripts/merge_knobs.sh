for t in 8 12 16; do for pe in 65536 32768 16384; do
echo "== threads $t part_elems $pe"
for c in w8a delicious; do echo -n "$c: "; HB_HOST_MERGE_THREADS=$t HB_MERGE_PART_ELEMS=$pe python scripts/e2e_probe3.py $c 2>&1 | grep -E "replica_step_host \(fused" | tr "\n" " " | sed "s/  */ /g"; echo; done
done; done
HB_DEBUG_XFER=1 HB_HOST_MERGE_THREADS=16 HB_MERGE_PART_ELEMS=32768 python scripts/xfer_host.py w8a 2>&1 | tail -12
