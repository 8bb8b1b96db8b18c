"""Host-side logic (no GPU): the logical KernelCounters the GPU path reports are the
reference's own (kernels.hpp:18-31, cost_model.hpp:44-154)."""
import ctypes as C

import numpy as np
import pytest

from oracle import bbsi_oracle as O
from oracle import ref_lib as R


def _lib_counters(l, levels):
    from paper_2605_19910_b200._native import lib

    out = np.zeros(3, dtype=np.int64)
    s2 = np.array(levels, dtype=np.int32)
    lib().bbsi_ddrgf_reference_counters(C.c_longlong(l), s2.ctypes.data_as(C.c_void_p), len(levels),
                                        out.ctypes.data_as(C.c_void_p))
    return tuple(int(x) for x in out)


@pytest.mark.parametrize("l,levels", [(10, [4]), (15, [4, 2]), (8, [1, 1, 1]), (18, [2]), (40, [4, 1]), (4096, [511]),
                                      (4096, [1023]), (2048, [255])])
def test_ddrgf_counters_match_closed_form(l, levels):
    if O.ddrgf_divides_evenly(l, levels):
        assert _lib_counters(l, levels) == O.predict_ddrgf_counters(l, levels).as_tuple()


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("l,levels", [(11, [4]), (12, [4]), (13, [4]), (6, [2, 1]), (15, [4, 1]), (40, [2, 1]),
                                      (21, [4, 2]), (10, [1])])
def test_ddrgf_counters_match_reference_uneven(l, levels):
    m = O.random_spd_like(O.make_layout(l, 2, 1), 17 + l, 2.0)
    _, c = R.ddrgf(m, levels)
    assert _lib_counters(l, levels) == c.as_tuple()
