"""The tcgen05 base conversion (bconv_t5_kernel) on its own, bit-exact against the oracle.

The fused pipelines call it with the ihat scale folded into the preceding INTT and
with lazy outputs; here it runs through the public `bc_convert` /
`bc_convert_centered` mirror (rnspoly.py:264-331), i.e. with the source pre-scale
and canonical outputs, on the shapes that exercise its chunking: one source,
K padding (9 sources -> 96 bytes), padded last chunk (23 targets), three chunks
(36 targets), four full chunks (64 targets), 16 sources (K = 128), and rings of
exactly one tile (N = 128) up to several CTAs.
"""

import numpy as np
import pytest

from oracle import ckks_np
from paper_2112_06396_b200 import rnspoly
from paper_2112_06396_b200.device import to_host
from paper_2112_06396_b200.params import prime_chain_below
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu

# (log2 N, sources, targets, source bits, target bits)
SHAPES = [
    (7, 1, 4, 50, 50),      # one tile, C1's digit shape
    (8, 3, 5, 54, 60),      # target count padded to a multiple of 4
    (10, 8, 24, 54, 54),    # C3 ModUp / ModDown shape: two chunks of 12
    (10, 9, 23, 60, 54),    # relinearisation ModDown: K padded to 96, last chunk padded
    (11, 9, 36, 50, 50),    # C5: three chunks
    (9, 16, 64, 54, 56),    # widest supported: K = 128, four chunks of 16
    (12, 8, 24, 60, 54),    # several CTAs
]


def _inputs(src, n, pattern, seed):
    rng = np.random.default_rng(seed)
    x = np.empty((len(src), n), dtype=np.uint64)
    for i, q in enumerate(src):
        if pattern == "random":
            x[i] = rng.integers(0, q, size=n, dtype=np.uint64)
        elif pattern == "max":
            x[i] = q - 1
        else:  # 0 / 1 / q-2 / q-1 cycling, shifted per limb
            cyc = np.array([q - 1, 0, 1, q - 2], dtype=np.uint64)
            x[i] = cyc[(np.arange(n) + i) % 4]
    return x


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "N2^%d_%dto%d_%d_%db" % s)
@pytest.mark.parametrize("pattern", ["random", "max", "mixed"])
def test_bconv_tensor_core(shape, pattern):
    logn, ns, nd, sbits, tbits = shape
    n = 1 << logn
    if sbits == tbits:
        allp, _ = prime_chain_below(n, sbits, ns + nd, sbits, 0)
        src, dst = allp[:ns], allp[ns:]
    else:
        src, dst = prime_chain_below(n, sbits, ns, tbits, nd)
    x = _inputs(src, n, pattern, 1000 * logn + ns)
    got = to_host(rnspoly.bc_convert(RnsPoly(src, x, "coeff"), dst).data)
    assert np.array_equal(got, ckks_np.bc_convert(x, src, dst))
    got = to_host(rnspoly.bc_convert_centered(RnsPoly(src, x, "coeff"), dst).data)
    assert np.array_equal(got, ckks_np.bc_convert_centered(x, src, dst))
