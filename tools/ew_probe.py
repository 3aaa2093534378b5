"""Device time of the elementwise add kernel on level-1550 polys at N=2^16 (10 polys cycled,
> L2), for A/B builds: HG_LIB_PATH=... python tools/ew_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib  # noqa: E402

for log_n in (16, 17):
    params = hg.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 5, device_rng=True)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    v = np.random.default_rng(2).uniform(-1, 1, params.slot_count)
    polys = [hg.mod_down(hg.encrypt_values(v, 45, pk, params, gen), 1550).c0 for _ in range(10)]
    ctx = _lib.get_context(log_n)
    for p in polys:
        p.add(polys[0])
    torch.cuda.synchronize()
    ctx.set_kernel_timing(True, kinds=("elementwise",))
    for r in range(50):
        polys[r % 10].add(polys[(r + 3) % 10])
    st = ctx.kernel_stats("elementwise")
    ctx.set_kernel_timing(False)
    us = st["ms"] * 1e3 / st["launches"]
    nbytes = 3 * params.n * 4 * 49
    print(f"N=2^{log_n} add: {us:.2f} us/launch, {nbytes / us / 1e3:.0f} GB/s")
