for nt in 0 1; do for pe in 1048576 4194304 32768; do
echo "=== NT $nt part_elems $pe"
for c in w8a delicious realsim scaled; do
echo -n "$c: "; HB_MERGE_NT=$nt HB_MERGE_PART_ELEMS=$pe HB_XCHG_MERGE=host python scripts/e2e_probe3.py $c 2>&1 | grep -E "replica_step" | tr '\n' ' ' | sed 's/  */ /g'; echo
done; done; done
