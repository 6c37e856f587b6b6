# A/B of the e2e leg: graph-replayed deferred calls + zero-copy small batches (new) vs eager deferred calls + DMA batches (old)
for c in covtype w8a delicious; do for i in 1 2; do
for mode in new old; do
  if [ $mode = old ]; then export HB_LAND_EAGER=1 HB_ZC_BATCH_MAX=0; else unset HB_LAND_EAGER HB_ZC_BATCH_MAX; fi
  timeout 300 python bench.py --config $c --skip-cpu --no-ttt --steps 50 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); e=d['e2e']; print('$c $mode e2e %.4e seq %.4e dev %.4e' % (e['value'], e['sequential']['value'], d['value']))"
done; done; done
