# covtype step time under the step knobs (device-timed, 50 steps)
for i in 1 2; do for v in NONE=1 HB_NO_FX_SPLIT=1 HB_SMALL_BN64=0 HB_NO_CONC_BWD=1 HB_NO_PDL=1 HB_DRAIN_KB_FWD=0 HB_DRAIN_KB_CRIT=2; do
  env $v timeout 300 python bench.py --config covtype --skip-cpu --no-ttt --skip-e2e --steps 50 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v ms/step %.4f' % d['ms_per_step'])"
done; done
