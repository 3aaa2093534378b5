"""cProfile of the cold setup's head at P17 (plan + hom_logreg + w / w^-1 / z: the part where the
host issues slower than the device retires), top entries by own and cumulative time.

    python tools/prof_logreg.py
"""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import gwas  # noqa: E402
from paper_1902_04303_b200.data import synth_gwas_dataset  # noqa: E402
from paper_1902_04303_b200.logreg import hom_logreg  # noqa: E402

params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
eng = hg.HeEngine(params, evk, rot)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
ds = synth_gwas_dataset(245, 4, 512, seed=0)
cfg = gwas.GwasConfig(n=245, d=4, k=512)
inputs = gwas.encrypt_gwas_inputs(ds, cfg, params, pk, gen, lazy_batches=True)
lr = inputs.logreg
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
gwas.plan_setup(eng, cfg.resolve(params))
beta, p_prev = hom_logreg(eng, lr, 3)
w = eng.mult(p_prev, eng.sub_from_const(1.0, p_prev))
w_inv = gwas.inverse_slots(eng, w, 3, 3.0)
z = gwas.compute_z(eng, lr.X, beta, lr.y, p_prev, w_inv)
th = time.perf_counter() - t
torch.cuda.synchronize()
pr.disable()
print(f"host issue {th:.3f}s wall {time.perf_counter() - t:.3f}s")
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(28)
    print(s.getvalue()[:7000])
