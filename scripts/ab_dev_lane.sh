# A/B of the e2e leg with and without the device lane (HB_NO_XCHG_DEVICE_LANE=1: every sole-writer layer on the
# mirror lane, so deferred calls replay the step graph)
for c in ${CONFIGS:-w8a delicious realsim}; do for i in 1 2; do for v in 0 1; do
  HB_NO_XCHG_DEVICE_LANE=$v timeout 400 python bench.py --config $c --skip-cpu --no-ttt --steps 50 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); e=d['e2e']; print('$c no_dev_lane=$v e2e %.4e seq %.4e dev %.4e' % (e['value'], e['sequential']['value'], d['value']))"
done; done; done
