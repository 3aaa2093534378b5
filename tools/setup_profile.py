"""Stage timings of the GWAS setup at P17 (config 0/3 shapes): where the 12 s go.

    python tools/setup_profile.py [--log-n 17] [--n 245]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib, gwas, matrix  # noqa: E402
from paper_1902_04303_b200.data import synth_gwas_dataset  # noqa: E402
from paper_1902_04303_b200.logreg import hom_logreg  # noqa: E402


class T:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.synchronize()
        self.t = time.time()
        self.l0 = _lib.total_launches()
        self.ops = hg.OpCounter()
        self.cm = hg.track_ops(self.ops)
        self.cm.__enter__()

    def __exit__(self, *a):
        self.cm.__exit__(*a)
        torch.cuda.synchronize()
        dt = time.time() - self.t
        print(f"{self.name:16s} {dt:7.2f}s launches {_lib.total_launches() - self.l0:7d} ops {self.ops.snapshot()}",
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-n", type=int, default=17)
    ap.add_argument("--n", type=int, default=245)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    params = hg.CkksParams(log_n=args.log_n, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    ds = synth_gwas_dataset(args.n, 4, 512, seed=0)
    cfg = gwas.GwasConfig(n=args.n, d=4, k=512)
    inputs = gwas.encrypt_gwas_inputs(ds, cfg, params, pk, gen, lazy_batches=True)
    for rep in range(args.reps):
        print(f"=== pass {rep} ===", flush=True)
        run_pass(eng, inputs)


def run_pass(eng, inputs):
    lr = inputs.logreg
    with T("hom_logreg"):
        beta, p_prev = hom_logreg(eng, lr, 3)
    with T("w"):
        w = eng.mult(p_prev, eng.sub_from_const(1.0, p_prev))
    with T("inverse"):
        w_inv = gwas.inverse_slots(eng, w, 3, 3.0)
    with T("compute_z"):
        z = gwas.compute_z(eng, lr.X, beta, lr.y, p_prev, w_inv)
    with T("hat=X XtXinv"):
        hat = matrix.cp_matmul(eng, lr.X, lr.XtX_inv)
    with T("cp_rep(hat,Xt)"):
        prod = matrix.cp_rep_matmul(eng, hat, lr.Xt_rep)
    with T("ccp_to_cp"):
        cols = matrix.ccp_to_cp(eng, prod)
    with T("identity_minus"):
        m = matrix.identity_minus(eng, cols, lr.X.rows)
    with T("z' = M z"):
        zp = gwas.orthogonalize_z(eng, m, z)
    with T("m_dup"):
        m_dup = matrix.duplicate_many(eng, m.cols, 256)
    print("levels: beta", beta.level_bits, "p", p_prev.level_bits, "w", w.level_bits, "w_inv", w_inv.level_bits,
          "z", z.level_bits, "M", m.cols[0].level_bits, "z'", zp.level_bits, "m_dup", m_dup[0].level_bits)


if __name__ == "__main__":
    main()
