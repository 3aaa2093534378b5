"""cProfile of one COLD config-3 setup at P17 (compute_setup incl. its plan), top entries by
own time: where the host time of the first pass goes.

    python tools/prof_setup.py [sort-key]
"""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import gwas  # noqa: E402
from paper_1902_04303_b200.data import synth_gwas_dataset  # noqa: E402

params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
eng = hg.HeEngine(params, evk, rot)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
ds = synth_gwas_dataset(245, 4, 512, seed=0)
inputs = gwas.encrypt_gwas_inputs(ds, gwas.GwasConfig(n=245, d=4, k=512), params, pk, gen, lazy_batches=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
out = gwas.compute_setup(eng, inputs)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(30)
print(s.getvalue()[:8000])
