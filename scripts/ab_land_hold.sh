# A/B of held write-backs (HB_LAND_HOLD: the lowest layers' D2H of a deferred call issued behind the next call's batch)
# (HB_LAND_HOLD was reverted after this measurement: DESIGN.md section 6 item 7)
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "land_async or fused_replica or pcie or concurrent or pipelined or host or small_net" 2>&1 | tail -2
for c in ${CONFIGS:-covtype scaled}; do for i in 1 2; do for h in 2 0 1; do
  HB_LAND_HOLD=$h timeout 400 python bench.py --config $c --skip-cpu --no-ttt --steps 30 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); e=d['e2e']; print('$c hold=$h e2e %.4e seq %.4e dev %.4e' % (e['value'], e['sequential']['value'], d['value']))"
done; done; done
