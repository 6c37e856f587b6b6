# split-K finish inside the GEMM (EPI_SPLIT_FIN, default) vs the separate splitk_epi kernel (HB_NO_FX_FIN=1):
# (EPI_SPLIT_FIN / HB_NO_FX_FIN were reverted after this measurement: bit-identical but 0.110 vs 0.092 ms/step)
# bit-identical losses / weights, and the covtype step time
python - <<'P'
import os, subprocess, sys, json
code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
import paper_2004_08771_b200 as hb
from oracle import ref_nn
out = []
for sizes, b in (((54, 512, 512, 512, 2), 512), ((37, 96, 3), 129), ((300, 256, 256, 4), 700), ((500, 1024, 1024, 983), 300)):
    w = ref_nn.init_weights(sizes, 3)
    x, _ = ref_nn.synthetic_blobs(b, sizes[0], 2, 2.5, 4)
    y = np.random.default_rng(5).integers(0, sizes[-1], b)
    ctx = hb.GpuReplica(sizes, b); ctx.set_weights(w); ctx.stage(x, y)
    ls = [ctx.step(0, b, 0.3, want_loss=True) for _ in range(3)]
    out.append((ls, [float(np.abs(a).sum()) for a in ctx.get_weights()], ctx.get_weights()))
    ctx.close()
np.save(sys.argv[1], np.array([o[2] for o in out], dtype=object), allow_pickle=True)
print([o[0][-1] for o in out])
'''
open("/tmp/fin_probe.py", "w").write(code)
a = subprocess.run([sys.executable, "/tmp/fin_probe.py", "/tmp/fin_on.npy"], capture_output=True, text=True)
b = subprocess.run([sys.executable, "/tmp/fin_probe.py", "/tmp/fin_off.npy"], capture_output=True, text=True, env={**os.environ, "HB_NO_FX_FIN": "1"})
print("on ", a.stdout.strip(), a.stderr[-300:])
print("off", b.stdout.strip(), b.stderr[-300:])
import numpy as np
A = np.load("/tmp/fin_on.npy", allow_pickle=True); B = np.load("/tmp/fin_off.npy", allow_pickle=True)
print("bit-identical weights:", all(np.array_equal(p, q) for ws, vs in zip(A, B) for p, q in zip(ws, vs)))
P
for i in 1 2; do for v in 0 1; do
  HB_NO_FX_FIN=$v timeout 300 python bench.py --config covtype --skip-cpu --no-ttt --skip-e2e --steps 50 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('HB_NO_FX_FIN=$v ms/step %.4f launches %d' % (d['ms_per_step'], d['gpu_launches']))"
done; done
