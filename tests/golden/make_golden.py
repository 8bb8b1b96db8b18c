"""Generates tests/golden/*.npz from the COMPILED, UNMODIFIED reference (oracle/_ref).

Run in a container that has /root/reference (python tests/golden/make_golden.py).
The fixtures pin the numpy oracle restatement (tests/test_oracle.py) where the
reference itself cannot run, e.g. on a GPU box without /root/reference sources.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import bbsi_oracle as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, m, **extra):
    lay = m.layout
    np.savez_compressed(OUT / f"{name}.npz", A=m.data, sizes=np.array(lay.block_sizes), w=lay.bandwidth, **extra)


def main():
    # test_rgf.cpp:34-40
    m = R.random_spd_like(O.make_layout(12, 8, 1), 77, 2.0)
    g, c = R.rgf_tridiag(m)
    save("rgf_tridiag_l12_b8_s77", m, G=g.data, counters=np.array(c.as_tuple()),
         dense=R.oracle_selected_inverse(m).data)
    # test_rgf.cpp:42-48 ragged
    m = R.random_spd_like(O.BlockLayout(5, [3, 1, 4, 2, 3], 1), 8, 2.0)
    g, c = R.rgf_tridiag(m)
    save("rgf_tridiag_ragged_s8", m, G=g.data, counters=np.array(c.as_tuple()))
    # test_rgf.cpp:58-67
    for w in (2, 3):
        m = R.random_spd_like(O.make_layout(10, 4, w), 100 + w, 2.0)
        tr = {}
        g, c = R.rgf_ndiag(m, tr)
        save(f"rgf_ndiag_l10_b4_w{w}", m, G=g.data, counters=np.array(c.as_tuple()),
             max_update_offset=tr["max_update_offset"])
    # test_rgf.cpp:79-88 fused
    m = R.random_spd_like(O.make_layout(9, 3, 2), 55, 2.0)
    g, c = R.rgf_fused(m)
    save("rgf_fused_l9_b3_w2", m, G=g.data, counters=np.array(c.as_tuple()))
    # test_rgf.cpp:97-123 extended
    m = R.random_spd_like(O.make_layout(5, 3, 1), 205, 2.0)
    e, c = R.rgf_extended(m)
    save("rgf_extended_l5_b3", m, G=e.core.data, counters=np.array(c.as_tuple()),
         first_row=np.array(e.first_row), last_row=np.array(e.last_row), first_col=np.array(e.first_col),
         last_col=np.array(e.last_col))
    # test_ddrgf.cpp:44-60 and trailing groups
    for l, lev in ((10, [4]), (15, [4, 2]), (13, [4]), (40, [2, 1])):
        m = R.random_spd_like(O.make_layout(l, 3, 1), 500 + l, 2.0)
        g, c = R.ddrgf(m, lev, 3)
        save(f"ddrgf_l{l}_b3_{'_'.join(map(str, lev))}", m, G=g.data, counters=np.array(c.as_tuple()),
             levels=np.array(lev))
    # test_rgf.cpp:150-160 Hermitian
    h = R.random_hermitian(O.make_layout(8, 3, 1), 31, 1.0)
    g, c = R.rgf_tridiag(h)
    save("hermitian_l8_b3_s31", h, G=g.data, counters=np.array(c.as_tuple()))
    # partition orders (test_partition.cpp:9-43)
    parts = {}
    for (l, s2) in ((10, 4), (11, 4), (12, 4), (2, 1)):
        order, inter, sep = R.interleave_permutation(l, 1, s2)
        parts[f"order_{l}_{s2}"] = np.array(order)
        parts[f"inter_{l}_{s2}"] = np.array(inter)
        parts[f"sep_{l}_{s2}"] = np.array(sep)
    np.savez_compressed(OUT / "partition_orders.npz", **parts)
    # .bbm files written by the reference io.cpp (test_io.cpp:22-38 shapes)
    m = R.random_spd_like(O.make_layout(5, 3, 2), 99, 2.0)
    m.data[0, 2, 0, 0] = complex(-0.0, 1e-308)
    R.write_bbm(OUT / "io_l5_b3_w2_s99.bbm", m)
    R.write_bbm(OUT / "io_ragged_l4_s123.bbm", R.random_spd_like(O.BlockLayout(4, [2, 5, 1, 3], 1), 123, 2.0))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
