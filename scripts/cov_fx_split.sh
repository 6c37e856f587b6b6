# covtype step time vs the cap on the forward / dX split-K count (HB_FX_SPLIT_MAX)
# (HB_FX_SPLIT_MAX was a temporary knob, reverted after this measurement)
for i in 1 2; do for v in 1000 2 3 4 6; do
  HB_FX_SPLIT_MAX=$v timeout 300 python bench.py --config covtype --skip-cpu --no-ttt --skip-e2e --steps 50 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('HB_FX_SPLIT_MAX=$v ms/step %.4f' % d['ms_per_step'])"
done; done
