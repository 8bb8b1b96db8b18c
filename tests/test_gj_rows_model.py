"""CPU: the numpy model of gj_rows_kernel's block algebra (tools/gj_rows_proto.py) --
two in-place Gauss-Jordan panels per step on all rows, raw pivot rows as the update's
right operand, one rank-2NB update, final row / column scatter -- inverts to rounding.
The CUDA kernel (csrc/zinv.cu) implements exactly these formulas; its own parity tests
are tests/test_gpu_kernels.py (reference tolerances: tests/test_dense_kernels.cpp:97-134)."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
import gj_rows_proto as P  # noqa: E402


@pytest.mark.parametrize("n", [32, 64, 160])
def test_block_algebra_inverts(n):
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    x = P.invert(a)
    ref = np.linalg.inv(a)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-12
    assert np.linalg.norm(a @ x - np.eye(n)) / np.sqrt(n) <= 1e-12


def test_pivot_rows_are_a_permutation():
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (96, 16)) + 1j * rng.uniform(-1, 1, (96, 16))
    src = P.gj_panel(a.copy(), np.ones(96, bool))
    assert len(set(src)) == 16
    # the eliminated panel holds the unit columns' row operation: E[:, P]; E M[:, K] = unit columns
    w = a.copy()
    src = P.gj_panel(w, np.ones(96, bool))
    e = np.eye(96, dtype=complex)
    e[:, src] = w
    unit = np.zeros((96, 16))
    unit[src, np.arange(16)] = 1
    assert np.abs(e @ a - unit).max() <= 1e-12
