"""CPU oracle: a numpy/scipy restatement of the reference bbsi solvers.

TEST INFRASTRUCTURE ONLY. Imported by tests/, by ``__graft_entry__.smoke()`` and by
``bench.py``'s cpu_baseline / reference arm, as the *checker*. The product path
(``paper_2605_19910_b200``) never imports this module.

Every function restates the reference algorithm it cites (paths relative to
``/root/reference/proj``). The dense kernels map one-to-one onto the LAPACK
routines the reference calls through LAPACKE/CBLAS (``core/include/bbsi/kernels.hpp``):
``zgetrf`` (scipy ``lu_factor``), ``zgetrs 'N'/'T'`` (scipy ``lu_solve``) and
``zgemm`` (numpy matmul). Pinned against the compiled reference (``oracle/_ref``)
and against the committed golden fixtures in ``tests/golden`` by
``tests/test_oracle.py``.

Band storage convention (shared with the product's Python mirror): a band is a
complex128 array ``band[a, off + w]`` of shape ``(l, 2w+1, bs, bs)``; block
``(a, a+off)`` occupies the top-left ``rows(a) x cols(a+off)`` corner, everything
else is zero. This is the reference's slot order (``block_banded.hpp:58-60``).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

EPS = np.finfo(np.float64).eps


# --------------------------------------------------------------------------- errors
class InvalidArgumentError(ValueError):
    """errors.hpp:9-12"""


class SingularMatrixError(RuntimeError):
    """errors.hpp:18-27: ``layer`` is the failing principal layer or -1."""

    def __init__(self, what: str, layer: int = -1):
        super().__init__(what)
        self.layer = layer


# --------------------------------------------------------------------------- counters
@dataclass
class KernelCounters:
    """kernels.hpp:18-31"""

    n_gemm: int = 0
    n_lu: int = 0
    n_getrs: int = 0

    def __iadd__(self, o):
        self.n_gemm += o.n_gemm
        self.n_lu += o.n_lu
        self.n_getrs += o.n_getrs
        return self

    def __add__(self, o):
        return KernelCounters(self.n_gemm + o.n_gemm, self.n_lu + o.n_lu, self.n_getrs + o.n_getrs)

    def as_tuple(self):
        return (self.n_gemm, self.n_lu, self.n_getrs)


def rgf_extra_gemms(l: int) -> int:
    """cost_model.hpp:44"""
    return 0 if l <= 2 else (l - 1) * (l - 2)


def predict_rgf_counters(l: int) -> KernelCounters:
    """cost_model.hpp:47-49"""
    return KernelCounters(4 * (l - 1), l, 3 * l - 2)


def predict_nrgf_counters(l: int, w: int) -> KernelCounters:
    """cost_model.hpp:52-54"""
    return KernelCounters((3 * w * w + w) * l - 2 * w**3 - 2 * w * w, l, l * (2 * w + 1) - w * w - w)


def predict_extended_counters(l: int) -> KernelCounters:
    """cost_model.hpp:57-61"""
    c = predict_rgf_counters(l)
    c.n_gemm += rgf_extra_gemms(l)
    return c


def ddrgf_divides_evenly(l: int, s2_levels) -> bool:
    """cost_model.hpp:126-133"""
    lk = l
    for s2 in s2_levels:
        if lk < 1 + s2 or lk % (1 + s2) != 0:
            return False
        lk //= 1 + s2
    return True


def predict_ddrgf_counters(l: int, s2_levels) -> KernelCounters:
    """cost_model.hpp:137-154"""
    c = KernelCounters()
    lk = l
    for s2 in s2_levels:
        if lk < 1 + s2:
            raise InvalidArgumentError("predict_ddrgf_counters: plan exhausts layers")
        n_tasks = (lk + s2) // (1 + s2)
        c.n_gemm += n_tasks * (4 * (s2 - 1) + rgf_extra_gemms(s2) + 2 * s2 + 2 * s2 + 4 + 4 * s2 + 4 + 6 * s2 - 4)
        c.n_lu += n_tasks * s2
        c.n_getrs += n_tasks * (3 * s2 - 2)
        lk = n_tasks
    return c + predict_rgf_counters(lk)


# --------------------------------------------------------------------------- layout
@dataclass
class BlockLayout:
    """layout.hpp:13-54"""

    num_layers: int
    block_sizes: list
    bandwidth: int

    def __post_init__(self):
        self.block_sizes = [int(b) for b in self.block_sizes]
        self.validate()

    def validate(self):
        if self.num_layers < 1:
            raise InvalidArgumentError("BlockLayout: num_layers must be >= 1")
        if len(self.block_sizes) != self.num_layers:
            raise InvalidArgumentError("BlockLayout: block_sizes length mismatch")
        if any(b < 1 for b in self.block_sizes):
            raise InvalidArgumentError("BlockLayout: block sizes must be >= 1")
        if self.bandwidth < 0:
            raise InvalidArgumentError("BlockLayout: negative bandwidth")
        if self.num_layers > 1 and self.bandwidth > self.num_layers - 1:
            raise InvalidArgumentError("BlockLayout: bandwidth exceeds num_layers - 1")
        if self.num_layers == 1 and self.bandwidth != 0:
            raise InvalidArgumentError("BlockLayout: single layer requires bandwidth 0")

    def total_dim(self):
        return sum(self.block_sizes)

    def uniform(self):
        return all(b == self.block_sizes[0] for b in self.block_sizes)

    def layer_offset(self, a):
        return sum(self.block_sizes[:a])

    @property
    def bs(self):
        return max(self.block_sizes)


def make_layout(num_layers, block_size, bandwidth):
    """layout.hpp:57-61"""
    if num_layers < 1 or block_size < 1:
        raise InvalidArgumentError("make_layout: dimensions must be >= 1")
    return BlockLayout(num_layers, [block_size] * num_layers, bandwidth)


class Band:
    """BlockBandedMatrix<complex<double>> (block_banded.hpp:15-64) in slot order."""

    def __init__(self, layout: BlockLayout, data: np.ndarray | None = None):
        self.layout = layout
        l, w, bs = layout.num_layers, layout.bandwidth, layout.bs
        if data is None:
            data = np.zeros((l, 2 * w + 1, bs, bs), dtype=np.complex128)
        self.data = data

    @property
    def num_layers(self):
        return self.layout.num_layers

    @property
    def bandwidth(self):
        return self.layout.bandwidth

    def in_band(self, a, off):
        l, w = self.layout.num_layers, self.layout.bandwidth
        return 0 <= a < l and abs(off) <= w and 0 <= a + off < l

    def block(self, a, off):
        if not self.in_band(a, off):
            raise InvalidArgumentError("BlockBandedMatrix: block outside band")
        r, c = self.layout.block_sizes[a], self.layout.block_sizes[a + off]
        return self.data[a, off + self.layout.bandwidth, :r, :c]

    def set_block(self, a, off, value):
        self.block(a, off)[...] = value

    def copy(self):
        return Band(self.layout, self.data.copy())


# --------------------------------------------------------------------------- generators
class MT19937_64:
    """std::mt19937_64 (raw 64-bit outputs), the engine behind UniformSource."""

    NN, MM = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [0] * self.NN
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self.NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.empty(0, dtype=np.uint64)
        self.pos = 0

    def _twist(self):
        mt = self.mt
        N, M = self.NN, self.MM
        one = np.uint64(1)

        def mix(hi, lo):
            x = (hi & self.UM) | (lo & self.LM)
            return (x >> one) ^ ((x & one) * self.MATRIX_A)

        # standard three-chunk vectorisation of the sequential twist
        old = mt.copy()
        mt[: N - M] = old[M:] ^ mix(old[: N - M], old[1 : N - M + 1])
        mt[N - M : N - 1] = mt[: M - 1] ^ mix(old[N - M : N - 1], old[N - M + 1 : N])
        mt[N - 1] = mt[M - 1] ^ mix(old[N - 1 : N], mt[0:1])[0]
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.buf = y
        self.pos = 0

    def take(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self.pos >= len(self.buf):
                self._twist()
            m = min(n - k, len(self.buf) - self.pos)
            out[k : k + m] = self.buf[self.pos : self.pos + m]
            self.pos += m
            k += m
        return out


class UniformSource:
    """detail::UniformSource (block_banded.hpp:70-91): raw bits -> [-1, 1)."""

    def __init__(self, seed: int):
        self.rng = MT19937_64(seed)

    def reals(self, n):
        return (self.rng.take(n) >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0

    def complexes(self, n):
        r = self.reals(2 * n)
        return r[0::2] + 1j * r[1::2]

    def block(self, rows, cols):
        """Column-major fill of a rows x cols complex block."""
        v = self.complexes(rows * cols)
        return v.reshape(cols, rows).T.copy()


def random_spd_like(layout: BlockLayout, seed: int, dominance: float) -> Band:
    """block_banded.hpp:99-133"""
    if not dominance > 0:
        raise InvalidArgumentError("random_spd_like: dominance must be positive")
    m = Band(layout)
    src = UniformSource(seed)
    w = layout.bandwidth
    for a in range(layout.num_layers):
        for off in range(-w, w + 1):
            if m.in_band(a, off):
                blk = m.block(a, off)
                blk[...] = src.block(*blk.shape)
    for a in range(layout.num_layers):
        diag = m.block(a, 0)
        for i in range(diag.shape[0]):
            row_sum = 0.0
            for off in range(-w, w + 1):
                if not m.in_band(a, off):
                    continue
                blk = m.block(a, off)
                for j in range(blk.shape[1]):
                    if off == 0 and j == i:
                        continue
                    row_sum += abs(blk[i, j])
            d = diag[i, i]
            mag = abs(d)
            # std::complex / complex(mag, 0) divides each component (libgcc __divdc3
            # with d = 0); numpy's complex/float would multiply by 1/mag instead.
            phase = complex(d.real / mag, d.imag / mag) if mag > 1e-12 else 1.0 + 0j
            diag[i, i] = d + phase * complex(dominance * row_sum, 0.0)
    return m


def random_hermitian(layout: BlockLayout, seed: int, dominance: float) -> Band:
    """tests/helpers.hpp:63-96"""
    h = Band(layout)
    src = UniformSource(seed)
    w = layout.bandwidth
    for a in range(layout.num_layers):
        for off in range(0, w + 1):
            if not h.in_band(a, off):
                continue
            blk = h.block(a, off)
            blk[...] = src.block(*blk.shape)
            if off == 0:
                sym = blk.conj().T + blk
                blk[...] = 0.5 * sym
            else:
                h.block(a + off, -off)[...] = blk.conj().T
    for a in range(layout.num_layers):
        diag = h.block(a, 0)
        for i in range(diag.shape[0]):
            row = 0.0
            for off in range(-w, w + 1):
                if not h.in_band(a, off):
                    continue
                blk = h.block(a, off)
                for j in range(blk.shape[1]):
                    if off != 0 or j != i:
                        row += abs(blk[i, j])
            diag[i, i] = diag[i, i].real + dominance * row + 1.0
    return h


# --------------------------------------------------------------------------- dense kernels
@dataclass
class LUFactors:
    """kernels.hpp:94-99 (scipy keeps LAPACK packed LU + 0-based pivots)."""

    lu: np.ndarray
    piv: np.ndarray
    dim: int


def lu_factor(a: np.ndarray, c: KernelCounters) -> LUFactors:
    """kernels.hpp:140-160: zgetrf + negligible-pivot threshold eps*n*max|A|."""
    if a.shape[0] != a.shape[1]:
        raise InvalidArgumentError("lu_factor: matrix not square")
    c.n_lu += 1
    n = a.shape[0]
    if n == 0:
        return LUFactors(a.copy(), np.zeros(0, dtype=np.int32), 0)
    scale = np.abs(a).max()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lu, piv = sla.lu_factor(a, check_finite=False)
    tol = EPS * n * scale
    d = np.abs(np.diag(lu))
    if np.any(d == 0):
        raise SingularMatrixError("lu_factor: exactly singular matrix")
    bad = np.nonzero(d <= tol)[0]
    if bad.size:
        raise SingularMatrixError(f"lu_factor: negligible pivot {int(bad[0])}")
    return LUFactors(lu, piv, n)


def solve_left(f: LUFactors, b: np.ndarray, c: KernelCounters) -> np.ndarray:
    """kernels.hpp:163-174: zgetrs 'N'."""
    c.n_getrs += 1
    if f.dim == 0 or b.shape[1] == 0:
        return b.copy()
    return sla.lu_solve((f.lu, f.piv), b, trans=0, check_finite=False)


def solve_right(b: np.ndarray, f: LUFactors, c: KernelCounters) -> np.ndarray:
    """kernels.hpp:178-189: B A^{-1} via zgetrs 'T' on B^T."""
    c.n_getrs += 1
    if f.dim == 0 or b.shape[0] == 0:
        return b.copy()
    return sla.lu_solve((f.lu, f.piv), b.T, trans=1, check_finite=False).T


def invert(f: LUFactors, c: KernelCounters) -> np.ndarray:
    """kernels.hpp:192-195"""
    return solve_left(f, np.eye(f.dim, dtype=np.complex128), c)


def gemm(alpha, a, b, beta, cmat, c: KernelCounters):
    """kernels.hpp:102-117 (gemm_into semantics; returns the new C)."""
    c.n_gemm += 1
    if cmat is None:
        return alpha * (a @ b)
    return alpha * (a @ b) + beta * cmat


def _lu_pivot(a, layer, c):
    """rgf.hpp:20-29"""
    try:
        return lu_factor(a, c)
    except SingularMatrixError as e:
        raise SingularMatrixError(f"singular Schur pivot at layer {layer}: {e}", layer) from None


# --------------------------------------------------------------------------- solvers
def rgf_tridiag(m: Band):
    """rgf.hpp:37-76. Returns (G band, counters)."""
    l = m.num_layers
    if m.bandwidth != 1 and l != 1:
        raise InvalidArgumentError("rgf_tridiag: requires bandwidth 1")
    c = KernelCounters()
    g = Band(m.layout)
    if l == 1:
        f = _lu_pivot(m.block(0, 0), 0, c)
        g.set_block(0, 0, invert(f, c))
        return g, c
    f = [None] * l
    umult = [None] * (l - 1)
    lmult = [None] * (l - 1)
    f[l - 1] = _lu_pivot(m.block(l - 1, 0), l - 1, c)
    for i in range(l - 2, -1, -1):
        umult[i] = solve_right(m.block(i, +1), f[i + 1], c)
        lmult[i] = solve_left(f[i + 1], m.block(i + 1, -1), c)
        pivot = gemm(-1, m.block(i, +1), lmult[i], 1, m.block(i, 0), c)
        f[i] = _lu_pivot(pivot, i, c)
    g.set_block(0, 0, invert(f[0], c))
    for i in range(1, l):
        g.set_block(i - 1, +1, gemm(-1, g.block(i - 1, 0), umult[i - 1], 0, None, c))
        g.set_block(i, -1, gemm(-1, lmult[i - 1], g.block(i - 1, 0), 0, None, c))
        gi = invert(f[i], c)
        g.set_block(i, 0, gemm(-1, lmult[i - 1], g.block(i - 1, +1), 1, gi, c))
    return g, c


def rgf_ndiag(m: Band, trace: dict | None = None):
    """rgf.hpp:82-137. ``trace['max_update_offset']`` mirrors StructuralTrace."""
    l, w = m.num_layers, m.bandwidth
    if w < 1 and l != 1:
        raise InvalidArgumentError("rgf_ndiag: requires bandwidth >= 1")
    if l == 1:
        return rgf_tridiag(m)
    c = KernelCounters()
    if trace is not None:
        trace["max_update_offset"] = 0
    mp = m.copy()
    f = [None] * l
    lm = [None] * l
    um = [None] * l
    for j in range(l - 1, 0, -1):
        k = min(w, j)
        f[j] = _lu_pivot(mp.block(j, 0), j, c)
        lm[j] = [None] * k
        um[j] = [None] * k
        for t in range(1, k + 1):
            lm[j][t - 1] = solve_left(f[j], mp.block(j, -t), c)
            um[j][t - 1] = solve_right(mp.block(j - t, +t), f[j], c)
        for s in range(1, k + 1):
            for t in range(1, k + 1):
                mp.set_block(j - s, s - t, gemm(-1, mp.block(j - s, +s), lm[j][t - 1], 1, mp.block(j - s, s - t), c))
                if trace is not None:
                    trace["max_update_offset"] = max(trace["max_update_offset"], abs(s - t))
    f[0] = _lu_pivot(mp.block(0, 0), 0, c)
    g = Band(m.layout)
    g.set_block(0, 0, invert(f[0], c))
    for j in range(1, l):
        k = min(w, j)
        for t in range(1, k + 1):
            acc = None
            for s in range(1, k + 1):
                acc = gemm(-1, lm[j][s - 1], g.block(j - s, s - t), 0 if s == 1 else 1, acc, c)
            g.set_block(j, -t, acc)
        for t in range(1, k + 1):
            acc = None
            for s in range(1, k + 1):
                acc = gemm(-1, g.block(j - t, t - s), um[j][s - 1], 0 if s == 1 else 1, acc, c)
            g.set_block(j - t, +t, acc)
        acc = invert(f[j], c)
        for s in range(1, k + 1):
            acc = gemm(-1, lm[j][s - 1], g.block(j - s, +s), 1, acc, c)
        g.set_block(j, 0, acc)
    return g, c


def rgf_fused(m: Band):
    """rgf.hpp:143-192"""
    l, w = m.num_layers, m.bandwidth
    if w < 1 and l != 1:
        raise InvalidArgumentError("rgf_fused: requires bandwidth >= 1")
    if not m.layout.uniform():
        raise InvalidArgumentError("rgf_fused: requires uniform block sizes")
    if w <= 1:
        return rgf_tridiag(m)
    lp = (l + w - 1) // w
    sizes = [sum(m.layout.block_sizes[s * w : min(l, s * w + w)]) for s in range(lp)]
    fl = BlockLayout(lp, sizes, 0 if lp == 1 else 1)
    fused = Band(fl)

    def loc(a):
        return sum(m.layout.block_sizes[(a // w) * w : a])

    for a in range(l):
        for off in range(-w, w + 1):
            if not m.in_band(a, off):
                continue
            b = a + off
            src = m.block(a, off)
            dst = fused.block(a // w, b // w - a // w)
            r0, c0 = loc(a), loc(b)
            dst[r0 : r0 + src.shape[0], c0 : c0 + src.shape[1]] = src
    gf, c = rgf_tridiag(fused)
    g = Band(m.layout)
    for a in range(l):
        for off in range(-w, w + 1):
            if not m.in_band(a, off):
                continue
            b = a + off
            src = gf.block(a // w, b // w - a // w)
            dst = g.block(a, off)
            r0, c0 = loc(a), loc(b)
            dst[...] = src[r0 : r0 + dst.shape[0], c0 : c0 + dst.shape[1]]
    return g, c


@dataclass
class ExtendedInverse:
    """rgf.hpp:197-204"""

    core: Band
    first_row: list = field(default_factory=list)
    last_row: list = field(default_factory=list)
    first_col: list = field(default_factory=list)
    last_col: list = field(default_factory=list)


def rgf_extended(m: Band):
    """rgf.hpp:209-270 (the O(l^2) halo of the reference, kept verbatim)."""
    l = m.num_layers
    if m.bandwidth != 1 and l != 1:
        raise InvalidArgumentError("rgf_extended: requires bandwidth 1")
    c = KernelCounters()
    g = Band(m.layout)
    ext = ExtendedInverse(g)
    if l == 1:
        f = _lu_pivot(m.block(0, 0), 0, c)
        g.set_block(0, 0, invert(f, c))
        b = g.block(0, 0).copy()
        ext.first_row = [b]
        ext.last_row = [b]
        ext.first_col = [b]
        ext.last_col = [b]
        return ext, c
    f = [None] * l
    umult = [None] * (l - 1)
    lmult = [None] * (l - 1)
    f[l - 1] = _lu_pivot(m.block(l - 1, 0), l - 1, c)
    for i in range(l - 2, -1, -1):
        umult[i] = solve_right(m.block(i, +1), f[i + 1], c)
        lmult[i] = solve_left(f[i + 1], m.block(i + 1, -1), c)
        pivot = gemm(-1, m.block(i, +1), lmult[i], 1, m.block(i, 0), c)
        f[i] = _lu_pivot(pivot, i, c)
    g.set_block(0, 0, invert(f[0], c))
    col = [None] * l
    row = [None] * l
    col[0] = row[0] = g.block(0, 0).copy()
    ext.first_row = [None] * l
    ext.first_col = [None] * l
    ext.first_row[0] = ext.first_col[0] = g.block(0, 0).copy()
    for j in range(1, l):
        g.set_block(j - 1, +1, gemm(-1, g.block(j - 1, 0), umult[j - 1], 0, None, c))
        g.set_block(j, -1, gemm(-1, lmult[j - 1], g.block(j - 1, 0), 0, None, c))
        gi = invert(f[j], c)
        g.set_block(j, 0, gemm(-1, lmult[j - 1], g.block(j - 1, +1), 1, gi, c))
        ncol = [None] * l
        nrow = [None] * l
        for a in range(0, j - 1):
            ncol[a] = gemm(-1, col[a], umult[j - 1], 0, None, c)
            nrow[a] = gemm(-1, lmult[j - 1], row[a], 0, None, c)
        ncol[j - 1] = g.block(j - 1, +1).copy()
        nrow[j - 1] = g.block(j, -1).copy()
        ncol[j] = nrow[j] = g.block(j, 0).copy()
        col, row = ncol, nrow
        ext.first_row[j] = col[0]
        ext.first_col[j] = row[0]
    ext.last_col = col[:l]
    ext.last_row = row[:l]
    return ext, c


# --------------------------------------------------------------------------- partition
@dataclass
class DomainDescriptor:
    """partition.hpp:16-34; groups are (first, count) tuples."""

    s1: int
    s2: int
    interior_groups: list
    separator_groups: list

    def n_tasks(self):
        return len(self.interior_groups)

    def num_separator_layers(self):
        return sum(cnt for _, cnt in self.separator_groups)


def interleave_permutation(layout: BlockLayout, s1: int, s2: int):
    """partition.hpp:39-75 -> (order, DomainDescriptor). ``order[p]`` = original layer."""
    if s1 < 1 or s2 < 1:
        raise InvalidArgumentError("interleave_permutation: s1, s2 must be >= 1")
    if layout.bandwidth != 1:
        raise InvalidArgumentError("interleave_permutation: requires bandwidth 1")
    l = layout.num_layers
    if l < s1 + s2:
        raise InvalidArgumentError("interleave_permutation: too few layers to split")
    interior, separator = [], []
    pos = 0
    while pos < l:
        rem = l - pos
        if rem >= s1 + s2:
            d2, d1 = s2, s1
        else:
            d1 = min(s1, rem)
            d2 = rem - d1
        interior.append((pos, d2))
        separator.append((pos + d2, d1))
        pos += d2 + d1
    order = [g0 + a for g0, cnt in separator for a in range(cnt)]
    order += [g0 + a for g0, cnt in interior for a in range(cnt)]
    return order, DomainDescriptor(s1, s2, interior, separator)


# --------------------------------------------------------------------------- ddrgf
def _zeros(bs):
    return np.zeros((bs, bs), dtype=np.complex128)


def compute_subdomain(m: Band, desc: DomainDescriptor, i: int):
    """ddrgf.hpp:85-140. Returns a dict mirroring SubdomainResult."""
    first, count = desc.interior_groups[i]
    r = {"task": i, "empty": count == 0, "counters": KernelCounters(), "counters_corr": KernelCounters()}
    if count == 0:
        return r
    bs = m.layout.block_sizes[0]
    c = r["counters"]
    sub = Band(BlockLayout(count, [bs] * count, 0 if count == 1 else 1))
    for a in range(count):
        for off in (-1, 0, 1):
            if sub.in_band(a, off):
                sub.set_block(a, off, m.block(first + a, off))
    try:
        ext, cext = rgf_extended(sub)
    except SingularMatrixError as e:
        glob = first + e.layer if e.layer >= 0 else -1
        raise SingularMatrixError(f"sub-domain {i}: singular pivot at layer {glob}", glob) from None
    r["ext"] = ext
    c += cext
    has_left = i > 0
    last = count - 1
    in_left = m.block(first - 1, +1) if has_left else _zeros(bs)
    out_left = m.block(first, -1) if has_left else _zeros(bs)
    in_right = m.block(first + count, -1)
    out_right = m.block(first + last, +1)
    r["v_left"] = [gemm(1, in_left, ext.first_row[a], 0, None, c) for a in range(count)]
    r["v_right"] = [None] * count
    r["w_left"] = [None] * count
    r["w_right"] = [None] * count
    # keep the reference's per-a interleaving of the four GEMMs (ddrgf.hpp:127-132)
    for a in range(count):
        r["v_right"][a] = gemm(1, in_right, ext.last_row[a], 0, None, c)
        r["w_left"][a] = gemm(1, ext.first_col[a], out_left, 0, None, c)
        r["w_right"][a] = gemm(1, ext.last_col[a], out_right, 0, None, c)
    w = [r["w_left"], r["w_right"]]
    su = [[None, None], [None, None]]
    for j2 in range(2):
        su[0][j2] = gemm(1, in_left, w[j2][0], 0, None, c)
        su[1][j2] = gemm(1, in_right, w[j2][last], 0, None, c)
    r["schur_update"] = su
    return r


def compute_subdomains(m: Band, desc: DomainDescriptor):
    """ddrgf.hpp:269-275"""
    return [compute_subdomain(m, desc, i) for i in range(desc.n_tasks())]


def assemble_schur(m: Band, order, desc: DomainDescriptor, results):
    """ddrgf.hpp:282-303 (separator quadrant of the permuted matrix minus updates)."""
    n1 = desc.num_separator_layers()
    seps = order[:n1]
    sizes = [m.layout.block_sizes[a] for a in seps]
    s = Band(BlockLayout(n1, sizes, 0 if n1 == 1 else 1))
    for j in range(n1):
        for off in (-1, 0, 1):
            if not s.in_band(j, off):
                continue
            a, b = seps[j], seps[j + off]
            if m.in_band(a, b - a):
                s.set_block(j, off, m.block(a, b - a))
    for r in results:
        if r["empty"]:
            continue
        sep = (r["task"] - 1, r["task"])
        for j1 in range(2):
            for j2 in range(2):
                if sep[j1] >= 0 and sep[j2] >= 0:
                    blk = s.block(sep[j1], sep[j2] - sep[j1])
                    blk -= r["schur_update"][j1][j2]
    return s


def _reduced_block(schur_inv: Band, j1, j2, bs):
    """ddrgf.hpp:75-79"""
    if j1 < 0 or j2 < 0 or not schur_inv.in_band(j1, j2 - j1):
        return _zeros(bs)
    return schur_inv.block(j1, j2 - j1)


def compute_y(r, schur_inv, desc, bs, c):
    """ddrgf.hpp:142-160"""
    count = desc.interior_groups[r["task"]][1]
    sep = (r["task"] - 1, r["task"])
    v = (r["v_left"], r["v_right"])
    ys = []
    for j2 in range(2):
        y = []
        for b in range(count):
            acc = None
            for j1 in range(2):
                acc = gemm(1, _reduced_block(schur_inv, sep[j2], sep[j1], bs), v[j1][b], 0 if j1 == 0 else 1, acc, c)
            y.append(acc)
        ys.append(y)
    r["y_left"], r["y_right"] = ys


def collect_separator_rows(r, desc, out):
    """ddrgf.hpp:164-174"""
    first, count = desc.interior_groups[r["task"]]
    if r["task"] > 0:
        out[(first - 1, first)] = -r["y_left"][0]
    out[(first + count, first + count - 1)] = -r["y_right"][count - 1]


def collect_separator_cols(r, schur_inv, desc, bs, out, c):
    """ddrgf.hpp:177-194"""
    first, count = desc.interior_groups[r["task"]]
    left, right = r["task"] - 1, r["task"]
    last = count - 1
    to_left = gemm(-1, r["w_left"][0], _reduced_block(schur_inv, left, left, bs), 0, None, c)
    to_left = gemm(-1, r["w_right"][0], _reduced_block(schur_inv, right, left, bs), 1, to_left, c)
    if r["task"] > 0:
        out[(first, first - 1)] = to_left
    to_right = gemm(-1, r["w_left"][last], _reduced_block(schur_inv, left, right, bs), 0, None, c)
    to_right = gemm(-1, r["w_right"][last], _reduced_block(schur_inv, right, right, bs), 1, to_right, c)
    out[(first + last, first + count)] = to_right


def diag_update_right(r, desc, c):
    """ddrgf.hpp:198-208"""
    count = desc.interior_groups[r["task"]][1]
    if len(r.get("y_left") or []) != count:
        raise InvalidArgumentError("correction_diag: separator_rows correction must run first")
    core = r["ext"].core
    for a in range(count):
        for b in range(max(0, a - 1), min(count - 1, a + 1) + 1):
            blk = core.block(a, b - a)
            blk[...] = gemm(1, r["w_left"][a], r["y_left"][b], 1, blk, c)
            blk[...] = gemm(1, r["w_right"][a], r["y_right"][b], 1, blk, c)


def diag_update_left(r, schur_inv, desc, bs, c):
    """ddrgf.hpp:212-235"""
    count = desc.interior_groups[r["task"]][1]
    sep = (r["task"] - 1, r["task"])
    w = (r["w_left"], r["w_right"])
    v = (r["v_left"], r["v_right"])
    z = []
    for j1 in range(2):
        zz = []
        for a in range(count):
            acc = None
            for j2 in range(2):
                acc = gemm(1, w[j2][a], _reduced_block(schur_inv, sep[j2], sep[j1], bs), 0 if j2 == 0 else 1, acc, c)
            zz.append(acc)
        z.append(zz)
    core = r["ext"].core
    for a in range(count):
        for b in range(max(0, a - 1), min(count - 1, a + 1) + 1):
            blk = core.block(a, b - a)
            for j1 in range(2):
                blk[...] = gemm(1, z[j1][a], v[j1][b], 1, blk, c)


def _ddrgf_level(m: Band, s2_levels, level: int):
    """ddrgf.hpp:344-412"""
    s2 = s2_levels[level]
    bs = m.layout.block_sizes[0]
    total = KernelCounters()
    order, desc = interleave_permutation(m.layout, 1, s2)
    n_tasks = desc.n_tasks()
    results = [compute_subdomain(m, desc, i) for i in range(n_tasks)]
    for r in results:
        total += r["counters"]
    schur = assemble_schur(m, order, desc, results)
    if level + 1 < len(s2_levels):
        if schur.num_layers < 1 + s2_levels[level + 1]:
            raise InvalidArgumentError(f"ddrgf: plan exhausts layers at level {level + 1}")
        schur_inv, ci = _ddrgf_level(schur, s2_levels, level + 1)
    else:
        schur_inv, ci = rgf_tridiag(schur)
    total += ci
    coupling = [dict() for _ in range(n_tasks)]
    for i, r in enumerate(results):
        if r["empty"]:
            continue
        cc = r["counters_corr"]
        compute_y(r, schur_inv, desc, bs, cc)
        collect_separator_rows(r, desc, coupling[i])
        collect_separator_cols(r, schur_inv, desc, bs, coupling[i], cc)
        diag_update_right(r, desc, cc)
    for r in results:
        total += r["counters_corr"]
    g = Band(m.layout)
    for j in range(schur_inv.num_layers):
        lj = desc.separator_groups[j][0]
        for off in (-1, 0, 1):
            if not schur_inv.in_band(j, off):
                continue
            lq = desc.separator_groups[j + off][0]
            if g.in_band(lj, lq - lj):
                g.set_block(lj, lq - lj, schur_inv.block(j, off))
    for r in results:
        if r["empty"]:
            continue
        first, count = desc.interior_groups[r["task"]]
        core = r["ext"].core
        for a in range(count):
            for off in (-1, 0, 1):
                if core.in_band(a, off):
                    g.set_block(first + a, off, core.block(a, off))
    for cset in coupling:
        for (ra, cb), blk in cset.items():
            g.set_block(ra, cb - ra, blk)
    return g, total


def ddrgf(m: Band, s2_levels, n_threads: int = 1, terminal_threads: int = 1):
    """ddrgf.hpp:420-428 (DomainPlan validation ddrgf.hpp:26-31)."""
    if len(s2_levels) == 0:
        raise InvalidArgumentError("DomainPlan: needs at least one level")
    if any(s < 1 for s in s2_levels):
        raise InvalidArgumentError("DomainPlan: s2 must be >= 1")
    if n_threads < 1 or terminal_threads < 1:
        raise InvalidArgumentError("DomainPlan: thread counts must be >= 1")
    if m.bandwidth != 1:
        raise InvalidArgumentError("ddrgf: requires bandwidth 1")
    if not m.layout.uniform():
        raise InvalidArgumentError("ddrgf: requires uniform block sizes")
    return _ddrgf_level(m, list(s2_levels), 0)


# --------------------------------------------------------------------------- dense oracle
def to_dense(m: Band) -> np.ndarray:
    """block_banded.hpp:136-151"""
    lay = m.layout
    n = lay.total_dim()
    d = np.zeros((n, n), dtype=np.complex128)
    for a in range(lay.num_layers):
        r0 = lay.layer_offset(a)
        for off in range(-lay.bandwidth, lay.bandwidth + 1):
            if not m.in_band(a, off):
                continue
            c0 = lay.layer_offset(a + off)
            blk = m.block(a, off)
            d[r0 : r0 + blk.shape[0], c0 : c0 + blk.shape[1]] = blk
    return d


def extract_bndiag(d: np.ndarray, layout: BlockLayout) -> Band:
    """block_banded.hpp:155-171"""
    out = Band(layout)
    for a in range(layout.num_layers):
        r0 = layout.layer_offset(a)
        for off in range(-layout.bandwidth, layout.bandwidth + 1):
            if not out.in_band(a, off):
                continue
            c0 = layout.layer_offset(a + off)
            blk = out.block(a, off)
            blk[...] = d[r0 : r0 + blk.shape[0], c0 : c0 + blk.shape[1]]
    return out


def oracle_selected_inverse(m: Band) -> Band:
    """block_banded.hpp:175-181"""
    c = KernelCounters()
    f = lu_factor(to_dense(m), c)
    return extract_bndiag(invert(f, c), m.layout)


# --------------------------------------------------------------------------- parity metric
def rel_frobenius_error(a: np.ndarray, ref: np.ndarray) -> float:
    """dense.hpp:121-128"""
    nref = np.linalg.norm(ref)
    nd = np.linalg.norm(a - ref)
    return float(nd / nref) if nref > 0 else float(nd)


def max_block_error(a: Band, b: Band) -> float:
    """tests/helpers.hpp:14-21"""
    e = 0.0
    for i in range(a.num_layers):
        for off in range(-a.bandwidth, a.bandwidth + 1):
            if a.in_band(i, off):
                e = max(e, rel_frobenius_error(a.block(i, off), b.block(i, off)))
    return e


def block_errors(a: Band, b: Band) -> np.ndarray:
    """All per-block relative Frobenius errors (for max / median reporting)."""
    out = []
    for i in range(a.num_layers):
        for off in range(-a.bandwidth, a.bandwidth + 1):
            if a.in_band(i, off):
                out.append(rel_frobenius_error(a.block(i, off), b.block(i, off)))
    return np.array(out)


def hermitian_defect(m: Band) -> float:
    """tests/helpers.hpp:98-107"""
    e = 0.0
    for a in range(m.num_layers):
        for off in range(-m.bandwidth, m.bandwidth + 1):
            if m.in_band(a, off):
                e = max(e, rel_frobenius_error(m.block(a, off), m.block(a + off, -off).conj().T))
    return e
