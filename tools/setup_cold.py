"""Cold GWAS setup at P17 (the whole-job's first pass): per-stage wall time with the host-side
first-use costs attributed — switching-key preparations (KeyCache misses), mask encodes
(host FFT waits) and torch allocator events (device mallocs, retries).

    python tools/setup_cold.py [--n 245]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib, ckks, gwas, matrix  # noqa: E402
from paper_1902_04303_b200.data import synth_gwas_dataset  # noqa: E402
from paper_1902_04303_b200.logreg import hom_logreg  # noqa: E402

BUSY = False
ACC = {"key_s": 0.0, "key_n": 0, "mask_s": 0.0, "mask_n": 0}


def _wrap_key_get():
    orig = ckks.KeyCache.get

    def get(self, key, level, big_l):
        m0 = self.misses
        t = time.perf_counter()
        r = orig(self, key, level, big_l)
        if self.misses != m0:
            ACC["key_s"] += time.perf_counter() - t
            ACC["key_n"] += 1
        return r
    ckks.KeyCache.get = get


def _wrap_mask():
    orig = ckks.HeEngine.mask

    def mask(self, spec, scale_bits=None):
        scale = scale_bits if scale_bits is not None else self.params.log_p_small
        hit = (spec, scale) in self._plaintext_cache
        t = time.perf_counter()
        r = orig(self, spec, scale_bits)
        if not hit:
            ACC["mask_s"] += time.perf_counter() - t
            ACC["mask_n"] += 1
        return r
    ckks.HeEngine.mask = mask


class T:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.synchronize()
        if BUSY:
            _lib.get_context(17).set_kernel_timing(True)
        self.acc = dict(ACC)
        torch.cuda.reset_peak_memory_stats()
        self.ms = torch.cuda.memory_stats()
        self.t = time.perf_counter()

    def __exit__(self, *a):
        th = time.perf_counter() - self.t
        torch.cuda.synchronize()
        dt = time.perf_counter() - self.t
        ms = torch.cuda.memory_stats()
        d = {k: ACC[k] - self.acc[k] for k in ACC}
        busy = ""
        if BUSY:
            ctx = _lib.get_context(17)
            st = {k: ctx.kernel_stats(k) for k in ("crt", "modup", "ntt", "pointwise", "elementwise")}
            ctx.set_kernel_timing(False)
            busy = "  device " + " ".join(f"{k} {v['ms']:.0f}ms/{v['launches']}" for k, v in st.items()) + \
                f" = {sum(v['ms'] for v in st.values()) / 1e3:.2f}s"
        print(f"{self.name:16s} wall {dt:6.2f}s (host issue {th:5.2f}s)  key-prep {d['key_n']:4d} "
              f"{d['key_s']:5.2f}s  masks {d['mask_n']:4d} {d['mask_s']:5.2f}s  "
              f"cudaMalloc {ms['num_device_alloc'] - self.ms.get('num_device_alloc', 0):5d} "
              f"retries {ms['num_alloc_retries'] - self.ms.get('num_alloc_retries', 0)} "
              f"reserved {ms['reserved_bytes.all.current'] / 1e9:5.1f} GB peak alloc "
              f"{ms['allocated_bytes.all.peak'] / 1e9:5.1f} GB{busy}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=245)
    ap.add_argument("--no-plan", action="store_true")
    ap.add_argument("--busy", action="store_true", help="per-stage device busy time by kernel class")
    args = ap.parse_args()
    global BUSY
    BUSY = args.busy
    _wrap_key_get()
    _wrap_mask()
    params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    ds = synth_gwas_dataset(args.n, 4, 512, seed=0)
    cfg = gwas.GwasConfig(n=args.n, d=4, k=512)
    inputs = gwas.encrypt_gwas_inputs(ds, cfg, params, pk, gen, lazy_batches=True)
    torch.cuda.synchronize()
    lr = inputs.logreg
    t0 = time.perf_counter()
    if not args.no_plan:
        with T("plan"):
            gwas.plan_setup(eng, cfg.resolve(params))
    with T("hom_logreg"):
        beta, p_prev = hom_logreg(eng, lr, 3)
    with T("w+inverse+z"):
        w = eng.mult(p_prev, eng.sub_from_const(1.0, p_prev))
        w_inv = gwas.inverse_slots(eng, w, 3, 3.0)
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
        gwas.orthogonalize_z(eng, m, z)
    with T("m_dup"):
        m_dup = matrix.duplicate_many(eng, m.cols, 256)
    with T("prepare"):
        m_dup = [eng.prepare(ct) for ct in m_dup]
    torch.cuda.synchronize()
    print(f"cold setup total {time.perf_counter() - t0:.2f}s  key cache {ckks.KEY_CACHE.bytes / 1e9:.1f} GB "
          f"({len(ckks.KEY_CACHE._lru)} keys)  launches {_lib.total_launches()}")


if __name__ == "__main__":
    main()
