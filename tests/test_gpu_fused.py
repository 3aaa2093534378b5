"""The fused kernels (pointwise products inside the inverse NTT, relinearise + add + rescale
inside the key switch's CRT epilogue) against the unfused kernel sequence, word for word, at
levels that exercise one and two CRT column jobs, word-aligned windows and both ring sizes.
Both arms also pass the oracle/golden parity tests; this one pins the fused epilogues' corner
cases (the cross-proxy race it once caught showed up in a handful of 8-coefficient groups)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_fused_matches_unfused(tmp_path):
    import fused_check

    for _ in range(2):   # repeat: races show up as run-to-run differences
        assert fused_check.compare(quick=True, workdir=str(tmp_path)) == 0
