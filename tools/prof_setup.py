import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd())
import torch
import paper_1902_04303_b200 as hg
from paper_1902_04303_b200 import gwas
from paper_1902_04303_b200.data import synth_gwas_dataset
params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
eng = hg.HeEngine(params, evk, rot)
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
ds = synth_gwas_dataset(245, 4, 512, seed=0)
inputs = gwas.encrypt_gwas_inputs(ds, gwas.GwasConfig(n=245, d=4, k=512), params, pk, gen, lazy_batches=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
out = gwas.compute_setup(eng, inputs)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
