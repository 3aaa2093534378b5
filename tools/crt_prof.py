"""Wait-cycle breakdown of the pipelined CRT kernel (diagnostic; needs a library built with
-DHG_CRT_PROF, loaded through HG_LIB_PATH):

    make -C exp/prof -f ../../paper_1902_04303_b200/csrc/Makefile ...   (see tools/crt_prof.sh)
    HG_LIB_PATH=exp/prof/libhegwas_b200.so python tools/crt_prof.py [--level 1550]

Prints, per role, the mean over CTAs of the cycles each warp spent waiting on each barrier,
as a fraction of the kernel's elapsed cycles, for the tensor CRT (3 outputs, shift 0) and the
fused key-switch CRT (2 outputs, window [L, L + l)) of one P17 ciphertext product.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib  # noqa: E402

ROLES = [("res TMA", [0], ["res_empty"]), ("MMA", [1], ["tm_empty", "a_full", "b_full"]),
         ("B TMA", [2], ["b_empty"]), ("convert", list(range(3, 11)), ["res_full", "a_empty", "store+fences", "v_combine"]),
         ("epilogue", list(range(11, 19)), ["hand_full", "add_full", "tm_full", "hand_empty", "tmem_ld", "-", "col_loop", "post"]),
         ("add TMA", [19], ["add_empty"])]


def read(lib):
    buf = (ctypes.c_ulonglong * (160 * 20 * 8))()
    assert lib.hg_crt_prof_read(buf) == 0
    return np.frombuffer(buf, dtype=np.uint64).reshape(160, 20, 8).astype(np.float64)


def report(name, t, nsm):
    t = t[:nsm]
    el = t[:, :, 5].max(axis=1).mean()
    print(f"{name}: elapsed {el:.0f} cycles (mean over {nsm} CTAs)")
    for role, warps, cats in ROLES:
        w = t[:, warps, :]
        if w[:, :, 5].max() == 0:
            continue
        parts = ", ".join(f"{c} {w[:, :, k].mean() / el:.2f}" for k, c in enumerate(cats) if c != "-")
        busy = 1 - sum(w[:, :, k].mean() for k in range(min(len(cats), 4))) / el
        print(f"  {role:9s} {parts}  | not waiting {busy:.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=1550)
    args = ap.parse_args()
    params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    vals = np.random.default_rng(0).uniform(-1, 1, params.slot_count)
    a = hg.mod_down(hg.encrypt_values(vals, 45, pk, params, gen), args.level)
    b = hg.mod_down(hg.encrypt_values(vals[::-1], 45, pk, params, gen), args.level)
    pa = eng.prepare(a)
    ctx = _lib.get_context(17)
    lib = ctx.lib
    lib.hg_crt_prof_read.restype = ctypes.c_int
    lib.hg_crt_prof_read.argtypes = [ctypes.c_void_p]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for _ in range(2):
        eng.mult(pa, b)
    torch.cuda.synchronize()
    # the last pipelined CRT launch of a product is the fused key switch
    eng.mult(pa, b)
    torch.cuda.synchronize()
    report("key-switch CRT (fused finish)", read(lib), nsm)
    # tensor only: hg_ct_prepare + the product's first CRT; run the tensor through hg_poly_tensor
    lvl = args.level
    ops = [x.operand(lvl) if hasattr(x, "operand") else None for x in (a.c0, a.c1, b.c0, b.c1)]
    outs = [torch.empty_like(a.c0.words) for _ in range(3)]
    o = [_lib.Operand(x.words.data_ptr(), lvl, 1) for x in (a.c0, a.c1, b.c0, b.c1)]
    del ops
    _lib.check(lib.hg_poly_tensor(ctx.handle, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), lvl,
                                  o[0], o[1], o[2], o[3], ctx.stream()))
    torch.cuda.synchronize()
    report("tensor CRT (3 outputs, unprescaled)", read(lib), nsm)


if __name__ == "__main__":
    main()
