"""Wait-cycle breakdown of the tcgen05 ModUp kernel (diagnostic; needs a library built with
-DHG_MODUP_PROF, loaded through HG_LIB_PATH):

    tools/exp_build.sh mprof -DHG_MODUP_PROF
    HG_LIB_PATH=exp/mprof/libhegwas_b200.so python tools/modup_prof.py

Prints, per role, the mean over CTAs of the cycles each warp spent waiting on each barrier (and
in the loaders' gather / the epilogue's column loop) as a fraction of the kernel's elapsed cycles:
for the ModUp of a fresh operand pair (prepare: 2 polys, tensor basis) and of the key switch's
input inside four batched products (4 polys, key-switch basis).
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib  # noqa: E402

LOADERS = int(os.environ.get("HG_MODUP_LOADERS", "8"))   # as the library was built
ROLES = [("B TMA", [0], ["b_empty"]), ("MMA", [1], ["a_full", "b_full", "tm_empty"]),
         ("loaders", list(range(2, 2 + LOADERS)), ["a_empty", "fl_empty", "gather+store"]),
         ("epilogue", list(range(2 + LOADERS, 18 + LOADERS)), ["fl_full", "tm_full", "col_loop"])]


def read(lib):
    buf = (ctypes.c_ulonglong * (160 * 32 * 8))()
    assert lib.hg_modup_prof_read(buf) == 0
    return np.frombuffer(buf, dtype=np.uint64).reshape(160, 32, 8).astype(np.float64)


def report(name, t, nsm):
    t = t[:nsm]
    el = t[:, :, 5].max(axis=1).mean()
    print(f"{name}: elapsed {el:.0f} cycles (mean over {nsm} CTAs)")
    for role, warps, cats in ROLES:
        w = t[:, warps, :]
        print(f"  {role:9s} " + ", ".join(f"{c} {w[:, :, k].mean() / el:.2f}" for k, c in enumerate(cats)))


def main():
    params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    vals = np.random.default_rng(0).uniform(-1, 1, params.slot_count)
    a = hg.mod_down(hg.encrypt_values(vals, 45, pk, params, gen), 1550)
    b = hg.mod_down(hg.encrypt_values(vals[::-1], 45, pk, params, gen), 1550)
    lib = _lib.load_library()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    preps = [eng.prepare(a) for _ in range(4)]
    torch.cuda.synchronize()
    eng.prepare(a)
    torch.cuda.synchronize()
    report("operand pair (prepare: 2 polys, level 1550)", read(lib), nsm)
    for _ in range(2):
        eng.mult_prepared_many(preps, [b] * 4)
    torch.cuda.synchronize()
    report("key-switch input of four products (4 polys)", read(lib), nsm)
    eng.rotate(a, 1)
    torch.cuda.synchronize()
    report("rotation (1 poly through the automorphism gather)", read(lib), nsm)


if __name__ == "__main__":
    main()
