"""cProfile of SnpBatchStream.start() at P17 (4 slots): the host cost of issuing a batch's uploads.

    python tools/prof_ring.py
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

params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
ds = synth_gwas_dataset(245, 4, 512, seed=0)
cfg = gwas.GwasConfig(n=245, d=4, k=512).resolve(params)
batch = gwas.build_snp_batch(ds.S, 0, cfg, params, pk, gen)
hb = gwas.HostSnpBatch.from_device(batch)
del batch
torch.cuda.synchronize()
for rep in range(2):
    stream = gwas.SnpBatchStream([hb] * 8, params, level=params.log_l - 150, slots=4)
    t = time.perf_counter()
    stream.allocate()
    t_alloc = time.perf_counter() - t
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    stream.start()
    th = time.perf_counter() - t
    pr.disable()
    torch.cuda.synchronize()
    print(f"pass {rep}: allocate {t_alloc:.3f}s, start() host {th:.3f}s, until uploaded {time.perf_counter() - t:.3f}s")
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14)
    print(s.getvalue()[:3500])
    del stream
