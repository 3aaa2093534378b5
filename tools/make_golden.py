"""Generate golden vectors by running the REFERENCE package (hegwas) in this container.

Outputs tests/golden/{unit_ops,deep_ops,gwas_toy}.npz.  Ring elements are stored in the
framework's limb-major layout ([W][N] uint32) under "<name>" with their modulus in
"<name>__bits".  The reference at /root/reference is imported read-only; it does not
exist on the GPU box, which is why these fixtures are committed.

    python tools/make_golden.py [unit|deep|gwas|all]
"""
from __future__ import annotations

import hashlib
import os
import random
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hegwas  # noqa: E402  (the reference)
from hegwas import ckks as rck  # noqa: E402
from hegwas.gwas import GwasConfig, compute_gwas_encrypted, decrypt_statistics, encrypt_gwas_inputs  # noqa: E402
from hegwas.oracle import CleartextDataset as RefDataset  # noqa: E402

from paper_1902_04303_b200.data import synth_gwas_dataset  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def words(coeffs, bits):
    w = (bits + 31) // 32
    mask = (1 << bits) - 1
    buf = b"".join((c & mask).to_bytes(4 * w, "little") for c in coeffs)
    return np.ascontiguousarray(np.frombuffer(buf, dtype="<u4").reshape(len(coeffs), w).T)


def key_hash(elem) -> str:
    return hashlib.sha256(words(elem.coeffs, elem.mod_bits).tobytes()).hexdigest()


class Store:
    def __init__(self):
        self.d = {}

    def ring(self, name, elem):
        self.d[name] = words(elem.coeffs, elem.mod_bits)
        self.d[name + "__bits"] = np.int64(elem.mod_bits)

    def ct(self, name, ct):
        self.ring(name + ".c0", ct.c0)
        self.ring(name + ".c1", ct.c1)
        self.d[name + ".meta"] = np.array([ct.level_bits, ct.scale_bits, ct.depth_ct, ct.depth_pt,
                                           {None: 0, "ct": 1, "pt": 2}[ct.pending]], dtype=np.int64)

    def arr(self, name, a):
        self.d[name] = np.asarray(a)

    def save(self, fname):
        path = os.path.join(OUT, fname)
        np.savez_compressed(path, **self.d)
        print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def params_arr(p):
    return np.array([p.log_n, p.log_l, p.log_p, p.log_p_small, p.h], dtype=np.int64)


def rand_vec(seed, slots, scale=1.0):
    rng = np.random.default_rng(seed)
    return scale * (rng.uniform(-1, 1, slots) + 1j * rng.uniform(-1, 1, slots))


def per_op_cases(st: Store, params, seed, full_keys: bool):
    t0 = time.time()
    sk, pk, evk, rot = hegwas.keygen(params, seed)
    print(f"  keygen {time.time() - t0:.1f}s")
    st.arr("params", params_arr(params))
    st.arr("key_seed", np.int64(seed))
    if full_keys:
        st.ring("sk.s", sk.s)
        st.ring("pk.b", pk.b)
        st.ring("pk.a", pk.a)
        st.ring("evk.b", evk.b)
        st.ring("evk.a", evk.a)
        for amt, (b, a) in rot.keys.items():
            st.ring(f"rot{amt}.b", b)
            st.ring(f"rot{amt}.a", a)
        st.ring("conj.b", rot.conj[0])
        st.ring("conj.a", rot.conj[1])
    hashes = {"sk.s": key_hash(sk.s), "pk.b": key_hash(pk.b), "pk.a": key_hash(pk.a),
              "evk.b": key_hash(evk.b), "evk.a": key_hash(evk.a),
              "conj.b": key_hash(rot.conj[0]), "conj.a": key_hash(rot.conj[1])}
    for amt, (b, a) in rot.keys.items():
        hashes[f"rot{amt}.b"] = key_hash(b)
        hashes[f"rot{amt}.a"] = key_hash(a)
    st.arr("key_hash_names", np.array(sorted(hashes)))
    st.arr("key_hash_values", np.array([hashes[k] for k in sorted(hashes)]))

    eng = hegwas.HeEngine(params, evk, rot)
    slots = params.slot_count
    va, vb = rand_vec(1, slots), rand_vec(2, slots)
    st.arr("vec_a", va)
    st.arr("vec_b", vb)
    a = hegwas.encrypt_values(va, params.log_p, pk, params, random.Random(11))
    b = hegwas.encrypt_values(vb, params.log_p, pk, params, random.Random(12))
    st.ct("ct_a", a)
    st.ct("ct_b", b)
    # encoding (host, must be bit-identical)
    mask = eng.mask(("slot", 3))
    st.ring("mask_slot3", mask.m)
    st.ring("encode_a", hegwas.encode(va, params.log_p, params).m)
    t0 = time.time()
    st.ct("mult_raw", hegwas.mult(a, b, evk))
    st.ct("eng_mult", eng.mult(a, b))
    print(f"  mult {time.time() - t0:.1f}s")
    st.ct("rescale30", hegwas.rescale(a, 30))
    st.ct("rot1", eng.rotate(a, 1))
    st.ct("rot5", eng.rotate(a, 5))
    st.ct("rotl3", eng.rotate_left(a, 3))
    st.ct("conj", eng.conjugate(a))
    st.ct("mult_plain_mask", eng.mult_plain(a, mask))
    st.ct("mult_const", eng.mult_const(a, 0.125))
    st.ct("add_const", eng.add_const(a, 0.5))
    st.ct("sub_from_const", eng.sub_from_const(2.0, a))
    st.ct("mult_int_m1", hegwas.mult_integer(a, -1))
    st.ct("mult_int_4", hegwas.mult_integer(a, 4))
    st.ct("mod_down", hegwas.mod_down(a, params.log_l - 150))
    em = eng.mult(a, b)
    st.ct("eng_add_aligned", eng.add(em, a))
    st.ct("eng_mult2", eng.mult(em, b))
    e0, e1 = rck._keyswitch(a.c1, (evk.b, evk.a), a.level_bits, params.log_l)
    st.ring("keyswitch.e0", e0)
    st.ring("keyswitch.e1", e1)
    st.ring("decrypt_eng_mult", hegwas.decrypt(em, sk).m)
    st.arr("decoded_eng_mult", hegwas.decrypt_values(em, sk))


def make_unit():
    st = Store()
    params = hegwas.CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)
    per_op_cases(st, params, 7, full_keys=True)
    st.save("unit_ops.npz")


def make_deep():
    st = Store()
    params = hegwas.CkksParams(log_n=9, log_l=1700, log_p=45, log_p_small=30, h=64)
    per_op_cases(st, params, 3, full_keys=False)
    st.save("deep_ops.npz")


def make_gwas(n=8, d=4, k=16, log_n=7, seed=0, key_seed=5, fname="gwas_toy.npz", complex_packing=True,
              tau=None):
    st = Store()
    st.arr("complex_packing", np.int64(1 if complex_packing else 0))
    st.arr("tau", np.int64(tau or 0))
    params = hegwas.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30, h=64)
    st.arr("params", params_arr(params))
    st.arr("shape", np.array([n, d, k, seed, key_seed], dtype=np.int64))
    ds = synth_gwas_dataset(n, d, k, seed=seed)
    st.arr("X", ds.X)
    st.arr("S", ds.S)
    st.arr("y", ds.y)
    t0 = time.time()
    sk, pk, evk, rot = hegwas.keygen(params, key_seed)
    hashes = {"sk.s": key_hash(sk.s), "evk.b": key_hash(evk.b), "evk.a": key_hash(evk.a),
              "pk.b": key_hash(pk.b), "pk.a": key_hash(pk.a)}
    st.arr("key_hash_names", np.array(sorted(hashes)))
    st.arr("key_hash_values", np.array([hashes[x] for x in sorted(hashes)]))
    print(f"  keygen {time.time() - t0:.1f}s")
    config = GwasConfig(n=n, d=d, k=k, complex_packing=complex_packing, tau=tau).resolve(params)
    ref_ds = RefDataset(X=ds.X, S=ds.S, y=ds.y)
    rng = random.Random(seed)
    t0 = time.time()
    enc = encrypt_gwas_inputs(ref_ds, config, params, pk, rng)
    print(f"  encrypt {time.time() - t0:.1f}s")
    for j, c in enumerate(enc.logreg.X.cols):
        st.ct(f"in.X{j}", c)
    for j, c in enumerate(enc.logreg.Xt_rep.rows_ct):
        st.ct(f"in.Xt{j}", c)
    for j, c in enumerate(enc.logreg.XtX_inv.cols):
        st.ct(f"in.XtXinv{j}", c)
    st.ct("in.y", enc.logreg.y)
    st.arr("n_batches", np.int64(len(enc.batches)))
    for bi, batch in enumerate(enc.batches):
        for j, c in enumerate(batch.S_packed.rows_ct):
            st.ct(f"in.b{bi}.S{j}", c)
    engine = hegwas.HeEngine(params, evk, rot)
    t0 = time.time()
    with hegwas.track_ops() as ops:
        out = compute_gwas_encrypted(engine, enc, cache=None)
    print(f"  compute {time.time() - t0:.1f}s ops={ops.snapshot()}")
    st.arr("op_counts", np.array([ops.snapshot()[f] for f in sorted(ops.snapshot())], dtype=np.int64))
    st.arr("op_count_names", np.array(sorted(ops.snapshot())))
    st.arr("rotation_amounts", np.array(ops.rotation_amounts, dtype=np.int64))
    st.ct("out.beta", out.beta)
    st.ct("out.p_prev", out.p_prev)
    inter = out.intermediates
    st.ct("out.w", inter.w)
    st.ct("out.w_inv", inter.w_inv)
    st.ct("out.z", inter.z)
    st.ct("out.z_prime", inter.z_prime)
    for j, c in enumerate(inter.M.cols):
        st.ct(f"out.M{j}", c)
    for bo in out.batch_outputs:
        st.ct(f"out.b{bo.index}.num", bo.num_ct)
        st.ct(f"out.b{bo.index}.den_even", bo.den_even_ct)
        if bo.den_odd_ct is not None:
            st.ct(f"out.b{bo.index}.den_odd", bo.den_odd_ct)
    num, den = decrypt_statistics(out.batch_outputs, config, params, sk)
    st.arr("num", num)
    st.arr("den", den)
    st.save(fname)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    os.makedirs(OUT, exist_ok=True)
    if which in ("unit", "all"):
        make_unit()
    if which in ("deep", "all"):
        make_deep()
    if which in ("gwas", "all"):
        make_gwas()
    if which in ("hegw", "all"):
        make_hegw()
    if which == "real":
        make_gwas(k=11, seed=2, key_seed=7, fname="gwas_toy_real.npz", complex_packing=False, tau=8)
    if which in ("ragged", "all"):
        # k not a multiple of tau (16 + 5 SNPs, the last complex column half empty), and the
        # real-packing variant (tau = 8: 8 + 3 SNPs)
        make_gwas(k=21, seed=1, key_seed=6, fname="gwas_toy_ragged.npz")
        make_gwas(k=11, seed=2, key_seed=7, fname="gwas_toy_real.npz", complex_packing=False, tau=8)


def make_hegw():
    """HEGW v1 bytes written by the reference's own serialize module (UNIT params)."""
    from hegwas import serialize as S

    st = Store()
    params = hegwas.CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)
    sk, pk, evk, rot = hegwas.keygen(params, 7)
    eng = hegwas.HeEngine(params, evk, rot)
    a = hegwas.encrypt_values(rand_vec(1, params.slot_count), params.log_p, pk, params, random.Random(11))
    m = eng.mult(a, a)
    blobs = {
        "ct_a": S.ciphertext_to_bytes(a),
        "ct_mult": S.ciphertext_to_bytes(m),
        "pt_mask": S.plaintext_to_bytes(eng.mask(("slot", 3)), params.log_n),
        "sk": S.secret_key_to_bytes(sk, params.log_n),
        "pk": S.public_key_to_bytes(pk, params.log_n),
        "evk": S.evaluation_key_to_bytes(evk, params.log_n),
        "rot": S.rotation_keys_to_bytes(rot, params.log_n),
    }
    for k, v in blobs.items():
        st.arr("hegw." + k, np.frombuffer(v, dtype=np.uint8))
    st.arr("params", params_arr(params))
    st.save("hegw_unit.npz")


if __name__ == "__main__":
    main()
