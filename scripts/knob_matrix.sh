# GPU parity suite under every A/B switch of the measured optimisations
# (README "Knobs"): each must stay parity-green, they only change speed.
for v in HB_NO_GRAPHS HB_NO_CONC_BWD HB_NO_PDL HB_NO_FX_SPLIT HB_NO_EXACT_X HB_SPLITK_FUSION HB_NO_MIRROR HB_NO_DW_FIRST HB_NO_LAYER_MERGE HB_LAND_EAGER; do
  echo "$v: $(env $v=1 timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k 'not baseline_size and not loss_curve' 2>&1 | tail -1)"
done
echo "HB_XCHG_MERGE=dma: $(HB_XCHG_MERGE=dma timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k 'not baseline_size and not loss_curve' 2>&1 | tail -1)"
echo "HB_MIRROR_LANE=0: $(HB_MIRROR_LANE=0 timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not baseline_size and not loss_curve" 2>&1 | tail -1)"
echo "HB_DRAIN_KB_CRIT=0: $(HB_DRAIN_KB_CRIT=0 timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not baseline_size and not loss_curve" 2>&1 | tail -1)"
echo "HB_ZC_BATCH_MAX=0: $(HB_ZC_BATCH_MAX=0 timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not baseline_size and not loss_curve" 2>&1 | tail -1)"
