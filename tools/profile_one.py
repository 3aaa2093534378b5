"""Run one scheme op at P17 inside a cudaProfilerStart/Stop window (for
`ncu --profile-from-start off`).

    python tools/profile_one.py --op mult --level 1550 [--log-n 17 --log-l 1700] [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="mult")
    ap.add_argument("--level", type=int, default=1550)
    ap.add_argument("--log-n", type=int, default=17)
    ap.add_argument("--log-l", type=int, default=1700)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    params = hg.CkksParams(log_n=args.log_n, log_l=args.log_l, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    vals = np.random.default_rng(0).uniform(-1, 1, params.slot_count)
    a = hg.mod_down(hg.encrypt_values(vals, 45, pk, params, gen), args.level)
    b = hg.mod_down(hg.encrypt_values(vals[::-1], 45, pk, params, gen), args.level)
    mask = eng.mask(("slot", 3))
    preps = [eng.prepare(a) for _ in range(4)]
    ops = {"mult": lambda: eng.mult(a, b), "rotate": lambda: eng.rotate(a, 1),
           "mult_plain": lambda: eng.mult_plain(a, mask),
           # the batch step's unit of work: four products with resident left operands
           "mult4": lambda: eng.mult_prepared_many(preps, [b] * 4)}
    fn = ops[args.op]
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(args.reps):
        fn()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done", args.op, args.level)


if __name__ == "__main__":
    main()
