"""Two ranks (one process each, gloo, both on cuda:0 -- the ranks never wait on each other's
kernels: every exchange is a host-staged collective between whole phases) run the sharded
encrypted GWAS on the reference's toy run with a ragged second batch (tests/golden/
gwas_toy_ragged.npz): the column-split setup with its all-gathers of z' partials, M and M_dup
(paper_1902_04303_b200/parallel.py), then one batch per rank, the results gathered to rank 0.
Every gathered ciphertext must equal the reference's (hegwas gwas.py:293-333) bit for bit."""
import os
import socket
import traceback

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1902_04303_b200 as hg
        from paper_1902_04303_b200.gwas import GwasConfig
        from paper_1902_04303_b200.parallel import compute_gwas_encrypted_sharded, gather_to_root
        from tests.golden_io import Golden
        from tests.gpu_helpers import assert_ct_equal, params_from
        from tests.test_gpu_pipeline import _golden_inputs

        g = Golden("gwas_toy_ragged")
        params = params_from(g)
        n, d, k, seed, key_seed = (int(x) for x in g.arr("shape"))
        sk, pk, evk, rot = hg.keygen(params, key_seed)
        config = GwasConfig(n=n, d=d, k=k, complex_packing=True).resolve(params)
        enc = _golden_inputs(g, params, config)
        outs, inter, beta, p_prev = compute_gwas_encrypted_sharded(hg.HeEngine(params, evk, rot), enc,
                                                                  rank, world)
        # the split setup reproduces the single-GPU intermediates on every rank
        assert_ct_equal(beta, g, "out.beta")
        for name in ("w", "w_inv", "z", "z_prime"):
            assert_ct_equal(getattr(inter, name), g, f"out.{name}")
        assert len(inter.M.cols) == n
        for j, c in enumerate(inter.M.cols):
            assert_ct_equal(c, g, f"out.M{j}")
        local = {o.index: {"num": o.num_ct.c0.numpy_words(), "num1": o.num_ct.c1.numpy_words(),
                           "ev": o.den_even_ct.c0.numpy_words(), "ev1": o.den_even_ct.c1.numpy_words(),
                           "od": o.den_odd_ct.c0.numpy_words(), "od1": o.den_odd_ct.c1.numpy_words()}
                 for o in outs}
        merged = gather_to_root(local, world)
        if rank == 0:
            import numpy as np

            assert sorted(merged) == list(range(int(g.arr("n_batches"))))
            for b, parts in merged.items():
                for key, name in (("num", "num.c0"), ("num1", "num.c1"), ("ev", "den_even.c0"),
                                  ("ev1", "den_even.c1"), ("od", "den_odd.c0"), ("od1", "den_odd.c1")):
                    want, _ = g.words(f"out.b{b}.{name}")
                    assert np.array_equal(parts[key], want), f"batch {b} {name}"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
        q.close()
        q.join_thread()
        os._exit(0)   # skip the interpreter's CUDA / gloo teardown (slow in spawned ranks)
    except Exception:
        q.put((rank, traceback.format_exc()))
        # a failed rank may leave its peer blocked in a collective: leave without teardown
        q.close()
        q.join_thread()
        os._exit(1)


def test_two_ranks_split_setup_and_batches_bit_exact():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=600) for _ in procs)
        for p in procs:
            p.join(timeout=60)
    finally:
        for p in procs:   # never leave a rank behind (pytest would wait for it at exit)
            if p.is_alive():
                p.kill()
                p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res
    assert all(p.exitcode == 0 for p in procs)
