"""Host checks of the integer arithmetic the binning kernels rely on."""

import numpy as np


def test_emission_row_formula_exact():
    """k_emit_balanced (u16 tile ids): the rect row of position j is
    floor((j + 0.5) * RN(1/w)) in fp32 with no correction step.  Exhaustive
    over every j < 2^16 for w <= 600 and a spread of wide rects up to 65535."""
    j = np.arange(1 << 16, dtype=np.uint32)
    jf = j.astype(np.float32) + np.float32(0.5)
    widths = list(range(1, 601)) + [1000, 1023, 1024, 4095, 4096, 8191, 12345, 32767, 32768, 65534, 65535]
    for w in widths:
        rw = np.float32(1.0) / np.float32(w)          # __frcp_rn
        row = (jf * rw).astype(np.uint32)             # fp32 product, truncation
        assert np.array_equal(row, j // np.uint32(w)), w
