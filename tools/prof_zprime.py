"""cProfile of the setup's z' = M z stage at P17 (the host-issue-bound part of the cold setup):
top entries by own time.

    python tools/prof_zprime.py
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
from paper_1902_04303_b200 import gwas, matrix  # noqa: E402
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
gwas.plan_setup(eng, cfg.resolve(params))
beta, p_prev = hom_logreg(eng, lr, 3)
w = eng.mult(p_prev, eng.sub_from_const(1.0, p_prev))
w_inv = gwas.inverse_slots(eng, w, 3, 3.0)
z = gwas.compute_z(eng, lr.X, beta, lr.y, p_prev, w_inv)
m = gwas.compute_M(eng, lr.X, lr.XtX_inv, lr.Xt_rep)
torch.cuda.synchronize()
for rep in range(2):   # second pass: warm (keys / masks / tables built)
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    zp = gwas.orthogonalize_z(eng, m, z)
    th = time.perf_counter() - t
    torch.cuda.synchronize()
    pr.disable()
    print(f"pass {rep}: host issue {th:.3f}s wall {time.perf_counter() - t:.3f}s")
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
    print(s.getvalue()[:6000])
