# A/B of the headline e2e: deferred calls replaying the step graph (default) vs launched eagerly (HB_LAND_EAGER=1)
for i in 1 2 3; do for v in 0 1; do
  HB_LAND_EAGER=$v timeout 400 python bench.py --config ${CONFIG:-scaled} --skip-cpu --no-ttt > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); e=d['e2e']; print('eager=$v e2e %.4e seq %.4e dev %.4e' % (e['value'], e['sequential']['value'], d['value']))"
done; done
