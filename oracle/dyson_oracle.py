"""Independent numpy restatement of the Dyson generator spec (csrc/dyson_gen.h).

TEST INFRASTRUCTURE ONLY. The reference has no Dyson generator (SURVEY.md
finding 5); BASELINE.json defines the construction in words and this is the
written-down spec both sides consume:

  u     = (mix64(mix64(seed) ^ ctr) >> 11) * 2^-52 - 1        in [-1, 1)
  ctr   = (a << 40) | ((off + 8) << 36) | (2k + c),  k = col*b + row, c = 0 re / 1 im
  H_aa  = (X + X^dagger) / 2,  X = u(a, 0)
  H_a,a+off = s_off u(a, off) (s_1 = 0.5, s_2 = 0.2),   H_a+off,a = H_a,a+off^dagger
  A(E)  = (E + i eta) I - H - Sigma,  Sigma_a = -0.5i I on the first/last w layers
"""
from __future__ import annotations

import numpy as np

from . import bbsi_oracle as O

M64 = 0xFFFFFFFFFFFFFFFF


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform_block(seed: int, a: int, off: int, b: int) -> np.ndarray:
    """u(a, off) as a (row, col) complex block."""
    sm = mix64(np.uint64(seed))
    k = np.arange(b * b, dtype=np.uint64)  # column-major entry index
    base = (np.uint64(a) << np.uint64(40)) | (np.uint64(off + 8) << np.uint64(36))
    re = (mix64(sm ^ (base | (np.uint64(2) * k))) >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    im = (mix64(sm ^ (base | (np.uint64(2) * k + np.uint64(1)))) >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    v = re + 1j * im
    return v.reshape(b, b).T  # [col, row] -> (row, col)


def hamiltonian(l: int, w: int, b: int, seed: int) -> O.Band:
    h = O.Band(O.make_layout(l, b, w))
    scale = {1: 0.5}
    for a in range(l):
        x = uniform_block(seed, a, 0, b)
        h.set_block(a, 0, 0.5 * (x + x.conj().T))
        for off in range(1, w + 1):
            if a + off < l:
                u = uniform_block(seed, a, off, b)
                s = scale.get(off, 0.2)
                blk = (s * u.real) + 1j * (s * u.imag)
                h.set_block(a, off, blk)
                h.set_block(a + off, -off, blk.conj().T)
    return h


def dyson_matrix(h: O.Band, z: complex, sigma_layers: int) -> O.Band:
    """A = z I - H - Sigma with the generator's fixed operation order on the diagonal."""
    m = O.Band(h.layout, -h.data)
    l = h.num_layers
    for a in range(l):
        sg = -0.5j if (a < sigma_layers or a >= l - sigma_layers) else 0j
        d = m.block(a, 0)
        hd = np.diag(h.block(a, 0))
        re = (z.real - hd.real) - sg.real
        im = (z.imag - hd.imag) - sg.imag
        idx = np.arange(d.shape[0])
        d[idx, idx] = re + 1j * im
    return m
