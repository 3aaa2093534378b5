"""BASELINE config 2 (homomorphic matrix layer) timings on one GPU: the reference's
Algorithms 1-8 at config-2 shapes and the GPU-only extras of matrix_ext (X^T W X, X^T v,
diagonal-method matvec, LS sigmoids of degree 3/5/7, Newton matrix inverse).  Device-timed
with CUDA events, inputs resident; decrypted results checked against float64 replays.

    python tools/config2_bench.py [--log-n 16] [--log-l 1700] > profiles/r1_config2.json
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import matrix as mx  # noqa: E402
from paper_1902_04303_b200 import matrix_ext as me  # noqa: E402
from paper_1902_04303_b200.logreg import sigmoid7  # noqa: E402


def timed(fn, reps=3):
    out = fn()   # warm (key preparation at this level, masks)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        out = fn()
    e.record()
    torch.cuda.synchronize()
    return out, s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--log-l", type=int, default=1700)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    params = hg.CkksParams(log_n=args.log_n, log_l=args.log_l, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    rs = np.random.default_rng(0)
    x = rs.standard_normal((245, 5))
    x[:, 0] = 1.0
    a55 = rs.standard_normal((5, 5))
    w = rs.uniform(0, 0.25, 245)
    v5 = rs.standard_normal(5)
    r245 = rs.uniform(-1, 1, 245)
    enc = lambda v: hg.encrypt_values(v, 45, pk, params, gen)  # noqa: E731
    xcp = mx.CPMatrix(cols=[enc(x[:, j]) for j in range(5)], rows=245, cols_logical=5)
    a55cp = mx.CPMatrix(cols=[enc(a55[:, j]) for j in range(5)], rows=5, cols_logical=5)
    wct, vct, rct = enc(w), enc(v5), enc(r245)
    dec = lambda ct: hg.decrypt_values(ct, sk).real  # noqa: E731
    rows = []

    def rec(op, ms, err, **kw):
        rows.append(dict(op=op, ms=round(ms, 3), max_abs_err_vs_replay=float(f"{err:.3g}"), **kw))
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)

    out, ms = timed(lambda: mx.cp_matvec(eng, xcp, vct), args.reps)
    rec("cp_matvec 245x5 (Alg. 2)", ms, np.max(np.abs(dec(out)[:245] - x @ v5)))
    out, ms = timed(lambda: mx.cp_matmul(eng, a55cp, a55cp), args.reps)
    rec("cp_matmul 5x5 (Alg. 3)", ms, np.max(np.abs(mx.unpack_cp(out, sk)[:5, :5] - a55 @ a55)))
    out, ms = timed(lambda: mx.rp_matvec(eng, mx.RPMatrix(rows_ct=xcp.cols, rows=5, cols_logical=245), rct),
                    args.reps)
    rec("rp_matvec X^T r (Alg. 6)", ms, np.max(np.abs(dec(out)[:5] - x.T @ r245)))
    out, ms = timed(lambda: mx.dot_prod(eng, xcp.cols[1], rct, 245), args.reps)
    rec("dot_prod (Alg. 5, rotate-and-sum)", ms, abs(dec(out)[0] - x[:, 1] @ r245))
    ccp = mx.CCPMatrix(ct=enc(np.tile(np.r_[r245, np.zeros(11)], 4)), col_size=256, num_cols=4)
    out, ms = timed(lambda: mx.col_sum(eng, ccp), args.reps)
    rec("col_sum 4 cols of 256 (Alg. 4)", ms, abs(dec(out)[0] - r245.sum()))
    out, ms = timed(lambda: me.xt_w_x(eng, xcp, wct), args.reps)
    xtwx = x.T @ np.diag(w) @ x
    rec("X^T W X 245x5 (extra)", ms, np.max(np.abs(mx.unpack_cp(out, sk)[:5, :5] - xtwx)))
    a_ct = out
    out, ms = timed(lambda: me.xt_vec(eng, xcp, rct), args.reps)
    rec("X^T (y - p) 245x5 (extra)", ms, np.max(np.abs(dec(out)[:5] - x.T @ r245)))
    diags, period = me.pack_diagonals(x, pk, params, gen)
    vper = enc(me.periodic_vector(v5, period, params.slot_count))
    out, ms = timed(lambda: me.diag_matvec(eng, diags, vper), args.reps)
    rec("diagonal-method X beta 245x5 (extra)", ms, np.max(np.abs(dec(out)[:245] - x @ v5)))
    vper5 = enc(me.periodic_vector(v5, 8, params.slot_count))
    out, ms = timed(lambda: me.diag_matvec_plain(eng, a55, vper5), args.reps)
    rec("diagonal-method 5x5 plaintext matrix (extra)", ms, np.max(np.abs(dec(out)[:5] - a55 @ v5)))
    xs = np.linspace(-8, 8, params.slot_count)
    xct = enc(xs)
    for deg in (3, 5, 7):
        out, ms = timed(lambda: me.sigmoid_poly(eng, xct, deg), args.reps)
        rec(f"sigmoid LS degree {deg} (extra)", ms,
            np.max(np.abs(dec(out) - me.sigmoid_poly_eval(xs, me.sigmoid_ls_coeffs(deg)))),
            fit_max_err=round(float(np.max(np.abs(me.sigmoid_poly_eval(xs, me.sigmoid_ls_coeffs(deg))
                                                    - 1 / (1 + np.exp(-xs))))), 4))
    out, ms = timed(lambda: sigmoid7(eng, xct), args.reps)
    rec("sigmoid7 (reference coefficients)", ms, 0.0)
    alpha = me.newton_alpha(245, 5)
    out, ms = timed(lambda: me.newton_inverse(eng, a_ct, alpha, 7), 1)
    inv = mx.unpack_cp(out, sk)[:5, :5]
    rec("Newton matrix inverse 5x5, 7 iterations (extra)", ms,
        np.max(np.abs(inv - me.newton_inverse_replay(xtwx, alpha, 7))),
        residual_vs_true_inverse=float(f"{np.linalg.norm(inv @ xtwx - np.eye(5)):.3g}"))
    print(json.dumps({"config": f"config 2 matrix layer, N=2^{args.log_n}, log_l={args.log_l}, log_p=45, "
                                f"log_p_small=30; X 245x5 N(0,1) + intercept, 5x5 N(0,1), W in (0,0.25)",
                      "timing": "CUDA events, resident inputs, mean of reps after one warm call",
                      "ops": rows}, indent=1))


if __name__ == "__main__":
    main()
