"""A/B check of the fused CRT finish and the prescaled CRT inputs: ct-mult (+rescale), rotation
and batched-rotation outputs with and without HG_NO_FUSE + HG_NO_PRESCALE.

    python tools/fused_check.py            # runs both arms in subprocesses and compares
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [(13, lv) for lv in range(140, 1701, 70)] + [(13, 1088), (13, 1152), (13, 1024), (12, 1550), (17, 1550)]
QUICK = [(13, 1120), (13, 1540), (13, 230), (12, 1550)]


def arm(path, cases=None):
    import numpy as np
    import torch

    import paper_1902_04303_b200 as hg

    out = {}
    for log_n, level in cases or CASES:
        params = hg.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30)
        sk, pk, evk, rot = hg.keygen(params, 3, device_rng=True)
        eng = hg.HeEngine(params, evk, rot)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(9)
        v = np.random.default_rng(1).uniform(-1, 1, params.slot_count)
        a = hg.mod_down(hg.encrypt_values(v, 45, pk, params, gen), level)
        b = hg.mod_down(hg.encrypt_values(v[::-1], 45, pk, params, gen), level)
        c = eng.mult(a, b)
        r = eng.rotate(a, 3)
        m0 = hg.ckks.mult(a, b, evk)                       # no rescale
        pc = eng.mult(eng.prepare(a), b)                   # resident left operand
        rm = eng.rotate_many([a, b, a], 5)                 # batched key switches
        out[f"{log_n}_{level}_c0"] = c.c0.words.cpu().numpy()
        out[f"{log_n}_{level}_c1"] = c.c1.words.cpu().numpy()
        out[f"{log_n}_{level}_r0"] = r.c0.words.cpu().numpy()
        out[f"{log_n}_{level}_m0"] = m0.c0.words.cpu().numpy()
        out[f"{log_n}_{level}_p1"] = pc.c1.words.cpu().numpy()
        for k, x in enumerate(rm):
            out[f"{log_n}_{level}_b{k}"] = torch.cat([x.c0.words, x.c1.words]).cpu().numpy()
    np.savez(path, **out)


def compare(quick=False, workdir="/tmp"):
    """Run both arms in subprocesses (HG_NO_FUSE is read once per process); returns the number
    of output arrays that differ."""
    import numpy as np

    env = dict(os.environ)
    extra = ["--quick"] if quick else []
    on_path, off_path = os.path.join(workdir, "fused_on.npz"), os.path.join(workdir, "fused_off.npz")
    subprocess.run([sys.executable, __file__, on_path] + extra, check=True, env=env)
    env["HG_NO_FUSE"] = "1"
    env["HG_NO_PRESCALE"] = "1"
    subprocess.run([sys.executable, __file__, off_path] + extra, check=True, env=env)
    on, off = np.load(on_path), np.load(off_path)
    bad = 0
    for k in off.files:
        d = on[k] != off[k]
        if d.any():
            bad += 1
            w, i = np.nonzero(d)
            cs = sorted(set(i.tolist()))
            runs, st = [], cs[0]
            for a, b in zip(cs, cs[1:] + [None]):
                if b != a + 1:
                    runs.append((st, a))
                    st = b
            print(f"MISMATCH {k}: {d.sum()} words differ; words {sorted(set(w.tolist()))} coeff runs {runs[:12]}")
            c = cs[0]
            print("   fused  ", [hex(x) for x in on[k][:, c][:6]], "...", [hex(x) for x in on[k][:, c][-3:]])
            print("   unfused", [hex(x) for x in off[k][:, c][:6]], "...", [hex(x) for x in off[k][:, c][-3:]])
        else:
            print(f"ok {k} {off[k].shape}")
    print("mismatching arrays:", bad)
    return bad


def main():
    if len(sys.argv) > 1 and sys.argv[1] != "--quick":
        arm(sys.argv[1], QUICK if "--quick" in sys.argv else None)
        return
    compare(quick="--quick" in sys.argv)


if __name__ == "__main__":
    main()
