"""Python mirror of the reference ``bbsi`` solver interface, executed on the GPU.

Same names, argument meaning and error behaviour as the reference C++ library
(``/root/reference/proj/core/include/bbsi``):

* :class:`BlockLayout`, :func:`make_layout`         -- layout.hpp:13-61
* :class:`BlockBandedMatrix`                          -- block_banded.hpp:15-64
* :class:`KernelCounters`                             -- kernels.hpp:18-31
* :func:`rgf_tridiag`, :func:`rgf_ndiag`, :func:`rgf_fused`, :func:`rgf_extended`
                                                      -- rgf.hpp:37-270
* :class:`DomainPlan`, :func:`ddrgf`                  -- ddrgf.hpp:18-32, 420-428
* :class:`InvalidArgumentError`, :class:`SingularMatrixError` -- errors.hpp:9-27

Every solve crosses the C ABI (include/bbsi_cuda.h) into sm_100a kernels; there is
no CPU path. Blocks are complex128 (real inputs are promoted, as the survey's
drop-in contract allows; float inputs are rejected).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from ._native import last_error, lib


class InvalidArgumentError(ValueError):
    """bbsi::invalid_argument_error (errors.hpp:9-12)."""


class SingularMatrixError(RuntimeError):
    """bbsi::singular_matrix_error (errors.hpp:18-27); ``layer`` = failing layer or -1."""

    def __init__(self, what: str, layer: int = -1):
        super().__init__(what)
        self.layer = layer


class CudaError(RuntimeError):
    """A CUDA failure inside the native library (BBSI_CUDA_ERROR / BBSI_OUT_OF_MEMORY)."""


def _raise(rc: int, fail_layer: int = -1):
    if rc == 0:
        return
    msg = last_error()
    if rc == 1:
        raise InvalidArgumentError(msg)
    if rc == 2:
        raise SingularMatrixError(msg, fail_layer)
    raise CudaError(f"bbsi_cuda error {rc}: {msg}")


@dataclass
class KernelCounters:
    """kernels.hpp:18-31 -- the reference's *logical* call counts for the solve."""

    n_gemm: int = 0
    n_lu: int = 0
    n_getrs: int = 0

    def __add__(self, o):
        return KernelCounters(self.n_gemm + o.n_gemm, self.n_lu + o.n_lu, self.n_getrs + o.n_getrs)

    def as_tuple(self):
        return (self.n_gemm, self.n_lu, self.n_getrs)


@dataclass
class BlockLayout:
    """layout.hpp:13-54 (validation identical)."""

    num_layers: int
    block_sizes: list
    bandwidth: int

    def __post_init__(self):
        self.block_sizes = [int(b) for b in self.block_sizes]
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
    def slot_size(self):
        return max(self.block_sizes)


def make_layout(num_layers: int, block_size: int, bandwidth: int) -> BlockLayout:
    """layout.hpp:57-61"""
    if num_layers < 1 or block_size < 1:
        raise InvalidArgumentError("make_layout: dimensions must be >= 1")
    return BlockLayout(num_layers, [block_size] * num_layers, bandwidth)


class BlockBandedMatrix:
    """block_banded.hpp:15-64 with numpy storage ``data[a, off + w]`` (slot order).

    ``data`` has shape ``(l, 2w+1, bs, bs)``, bs = max block size; block ``(a, a+off)``
    is the top-left ``rows x cols`` corner of its slot.
    """

    def __init__(self, layout: BlockLayout, data: np.ndarray | None = None):
        self.layout = layout
        l, w, bs = layout.num_layers, layout.bandwidth, layout.slot_size
        if data is None:
            data = np.zeros((l, 2 * w + 1, bs, bs), dtype=np.complex128)
        else:
            data = np.asarray(data)
            if data.dtype in (np.float32, np.complex64):
                raise InvalidArgumentError("bbsi GPU path computes in complex128 only")
            data = data.astype(np.complex128, copy=False)
            if data.shape != (l, 2 * w + 1, bs, bs):
                raise InvalidArgumentError("BlockBandedMatrix: storage shape mismatch")
        self.data = data

    @property
    def num_layers(self):
        return self.layout.num_layers

    @property
    def bandwidth(self):
        return self.layout.bandwidth

    def in_band(self, a: int, off: int) -> bool:
        l, w = self.layout.num_layers, self.layout.bandwidth
        return 0 <= a < l and abs(off) <= w and 0 <= a + off < l

    def block(self, a: int, off: int) -> np.ndarray:
        if not self.in_band(a, off):
            raise InvalidArgumentError("BlockBandedMatrix: block outside band")
        r, c = self.layout.block_sizes[a], self.layout.block_sizes[a + off]
        return self.data[a, off + self.layout.bandwidth, :r, :c]

    def copy(self):
        return BlockBandedMatrix(self.layout, self.data.copy())

    # C ABI slot memory: column-major blocks
    def _slots(self) -> np.ndarray:
        return np.ascontiguousarray(self.data.transpose(0, 1, 3, 2))

    @classmethod
    def _from_slots(cls, layout, mem):
        return cls(layout, np.ascontiguousarray(mem.transpose(0, 1, 3, 2)))


@dataclass
class DomainPlan:
    """ddrgf.hpp:18-32"""

    s2_levels: list = field(default_factory=list)
    n_threads: int = 1
    terminal_threads: int = 1

    def n_levels(self):
        return len(self.s2_levels)

    def validate(self):
        if not self.s2_levels:
            raise InvalidArgumentError("DomainPlan: needs at least one level")
        if any(s < 1 for s in self.s2_levels):
            raise InvalidArgumentError("DomainPlan: s2 must be >= 1")
        if self.n_threads < 1 or self.terminal_threads < 1:
            raise InvalidArgumentError("DomainPlan: thread counts must be >= 1")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _args(m: BlockBandedMatrix):
    lay = m.layout
    sizes = np.array(lay.block_sizes, dtype=np.int32)
    a = m._slots()
    g = np.zeros_like(a)
    return lay, sizes, a, g


def rgf_tridiag(m: BlockBandedMatrix, trace: dict | None = None):
    """rgf.hpp:37-76 on the GPU. Returns (G, KernelCounters)."""
    lay, sizes, a, g = _args(m)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    rc = lib().bbsi_cuda_rgf_tridiag_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a), _ptr(g),
                                       _ptr(cnt), C.byref(fail))
    _raise(rc, fail.value)
    if trace is not None:
        trace["max_update_offset"] = 0
    return BlockBandedMatrix._from_slots(lay, g), KernelCounters(*map(int, cnt))


def rgf_many(ms: list) -> list:
    """rgf_tridiag / rgf_ndiag (rgf.hpp:37-137) of many matrices of one layout in one device
    pass (bbsi_cuda_rgf_many_z). Returns [(G, KernelCounters)]; raises SingularMatrixError
    for the first matrix (in list order) with a negligible pivot, as calling the single
    solver on each in turn would."""
    if not ms:
        return []
    lay = ms[0].layout
    l, w, bs = lay.num_layers, lay.bandwidth, lay.slot_size
    for m in ms:
        if (m.layout.num_layers, m.layout.bandwidth, tuple(m.layout.block_sizes)) != (l, w, tuple(lay.block_sizes)):
            raise InvalidArgumentError("rgf_many: every matrix must have the same layout")
    sizes = np.array(lay.block_sizes, dtype=np.int32)
    a = np.ascontiguousarray(np.stack([_args(m)[2] for m in ms]))
    g = np.zeros_like(a)
    cnt = np.zeros(3, dtype=np.int64)
    fails = np.full(len(ms), -1, dtype=np.int32)
    rc = lib().bbsi_cuda_rgf_many_z(l, w, bs, _ptr(sizes), len(ms), _ptr(a), _ptr(g), _ptr(cnt), _ptr(fails))
    if rc == 2:
        k = int(np.argmax(fails >= 0))
        raise SingularMatrixError(f"singular Schur pivot at layer {int(fails[k])} (matrix {k})", int(fails[k]))
    _raise(rc)
    c = KernelCounters(*map(int, cnt))
    return [(BlockBandedMatrix._from_slots(lay, g[k]), c) for k in range(len(ms))]


def rgf_ndiag(m: BlockBandedMatrix, trace: dict | None = None):
    """rgf.hpp:82-137 on the GPU; ``trace`` mirrors StructuralTrace (rgf.hpp:14-16)."""
    lay, sizes, a, g = _args(m)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    mo = C.c_int(trace.get("max_update_offset", 0) if trace is not None else 0)
    rc = lib().bbsi_cuda_rgf_ndiag_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a), _ptr(g),
                                     _ptr(cnt), C.byref(mo), C.byref(fail))
    _raise(rc, fail.value)
    if trace is not None:
        trace["max_update_offset"] = mo.value
    return BlockBandedMatrix._from_slots(lay, g), KernelCounters(*map(int, cnt))


def rgf_fused(m: BlockBandedMatrix):
    """rgf.hpp:143-192 on the GPU."""
    lay, sizes, a, g = _args(m)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    rc = lib().bbsi_cuda_rgf_fused_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a), _ptr(g),
                                     _ptr(cnt), C.byref(fail))
    _raise(rc, fail.value)
    return BlockBandedMatrix._from_slots(lay, g), KernelCounters(*map(int, cnt))


@dataclass
class ExtendedInverse:
    """rgf.hpp:197-204"""

    core: BlockBandedMatrix
    first_row: list
    last_row: list
    first_col: list
    last_col: list


def rgf_extended(m: BlockBandedMatrix):
    """rgf.hpp:209-270 on the GPU (halos by O(l) recurrences)."""
    lay, sizes, a, g = _args(m)
    l, bs = lay.num_layers, lay.slot_size
    halos = [np.zeros((l, bs, bs), dtype=np.complex128) for _ in range(4)]
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    rc = lib().bbsi_cuda_rgf_extended_z(l, lay.bandwidth, bs, _ptr(sizes), _ptr(a), _ptr(g),
                                        *[_ptr(h) for h in halos], _ptr(cnt), C.byref(fail))
    _raise(rc, fail.value)
    bsz = lay.block_sizes
    fr, lr, fc, lc = [[h[k].T for k in range(l)] for h in halos]
    return (ExtendedInverse(BlockBandedMatrix._from_slots(lay, g),
                            [fr[k][: bsz[0], : bsz[k]].copy() for k in range(l)],
                            [lr[k][: bsz[-1], : bsz[k]].copy() for k in range(l)],
                            [fc[k][: bsz[k], : bsz[0]].copy() for k in range(l)],
                            [lc[k][: bsz[k], : bsz[-1]].copy() for k in range(l)]),
            KernelCounters(*map(int, cnt)))


def ddrgf(m: BlockBandedMatrix, plan: DomainPlan, ngpu: int | None = None):
    """ddrgf.hpp:420-428 on the GPU (stabilised DDRGF). ngpu > 1 shards the
    domains over GPUs 0..ngpu-1 of this process (bbsi_cuda_ddrgf_multi_z: NCCL all-gather
    of the interface packets); default: $BBSI_GPUS or 1."""
    plan.validate()
    if ngpu is None:
        ngpu = max(1, int(os.environ.get("BBSI_GPUS", "1")))
    lay, sizes, a, g = _args(m)
    s2 = np.array(plan.s2_levels, dtype=np.int32)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    if ngpu > 1:
        rc = lib().bbsi_cuda_ddrgf_multi_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a),
                                           _ptr(s2), len(s2), plan.n_threads, plan.terminal_threads, ngpu, None,
                                           _ptr(g), _ptr(cnt), C.byref(fail))
    else:
        rc = lib().bbsi_cuda_ddrgf_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a), _ptr(s2),
                                     len(s2), plan.n_threads, plan.terminal_threads, _ptr(g), _ptr(cnt),
                                     C.byref(fail))
    _raise(rc, fail.value)
    return BlockBandedMatrix._from_slots(lay, g), KernelCounters(*map(int, cnt))


def ddrgf_slots(A, G, l: int, bs: int, s2_levels, n_threads: int = 1, terminal_threads: int = 1):
    """ddrgf on raw slot memory (the C ABI's layout, w = 1): A, G complex128 (l, 3, bs, bs),
    C-contiguous host buffers (pinned for full PCIe rate). Raises like ddrgf()."""
    for name, x in (("A", A), ("G", G)):
        if not (isinstance(x, np.ndarray) and x.dtype == np.complex128 and x.shape == (l, 3, bs, bs)
                and x.flags.c_contiguous):
            raise InvalidArgumentError(f"{name}: expected a C-contiguous complex128 array of shape {(l, 3, bs, bs)}")
    s2 = np.array(list(s2_levels), dtype=np.int32)
    fail = C.c_int(-1)
    rc = lib().bbsi_cuda_ddrgf_z(l, 1, bs, None, _ptr(A), _ptr(s2), len(s2), n_threads, terminal_threads, _ptr(G),
                                 None, C.byref(fail))
    _raise(rc, fail.value)
    return G


def random_spd_like(layout: BlockLayout, seed: int, dominance: float) -> BlockBandedMatrix:
    """block_banded.hpp:99-133 (raw mt19937_64 stream of block_banded.hpp:70-91), generated
    host-side by the C ABI (bbsi_random_spd_like_z) in the reference's draw order."""
    sizes = np.array(layout.block_sizes, dtype=np.int32)
    l, w, bs = layout.num_layers, layout.bandwidth, layout.slot_size
    mem = np.zeros((l, 2 * w + 1, bs, bs), dtype=np.complex128)
    _raise(lib().bbsi_random_spd_like_z(l, w, bs, _ptr(sizes), C.c_uint64(seed), float(dominance), _ptr(mem)))
    return BlockBandedMatrix._from_slots(layout, mem)


# ------------------------------------------------------------------ .bbm files (io.cpp:26-75)
# One JSON header line {"version": 1, "num_layers", "block_sizes", "bandwidth",
# "scalar": "c128"}, then every in-band block (layer ascending, offset ascending),
# column-major, (re, im) little-endian float64 pairs.

def _inband(layout: BlockLayout):
    l, w = layout.num_layers, layout.bandwidth
    for a in range(l):
        for off in range(-w, w + 1):
            if 0 <= a + off < l:
                yield a, off


def write_bbm(path: str, m: BlockBandedMatrix) -> None:
    """io.cpp:26-45"""
    import json

    lay = m.layout
    header = {"version": 1, "num_layers": lay.num_layers, "block_sizes": lay.block_sizes,
              "bandwidth": lay.bandwidth, "scalar": "c128"}
    try:
        f = open(path, "wb")
    except OSError:
        raise InvalidArgumentError(f"write_bbm: cannot open {path}") from None
    with f:
        f.write((json.dumps(header, separators=(",", ":"), sort_keys=True) + "\n").encode())  # nlohmann dump order
        for a, off in _inband(lay):
            f.write(np.asarray(m.block(a, off), dtype="<c16").tobytes(order="F"))


def read_bbm(path: str) -> BlockBandedMatrix:
    """io.cpp:47-73 (same rejections: missing file, malformed header, version, scalar,
    truncated payload)."""
    import json

    try:
        f = open(path, "rb")
    except OSError:
        raise InvalidArgumentError(f"read_bbm: cannot open {path}") from None
    with f:
        line = f.readline()
        if not line:
            raise InvalidArgumentError("read_bbm: missing header")
        try:
            header = json.loads(line)
        except ValueError:
            header = None
        if not isinstance(header, dict):
            raise InvalidArgumentError("read_bbm: malformed header")
        if header.get("version", 0) != 1:
            raise InvalidArgumentError("read_bbm: unsupported version")
        if header.get("scalar", "") != "c128":
            raise InvalidArgumentError("read_bbm: unsupported scalar type")
        try:
            lay = BlockLayout(int(header["num_layers"]), list(header["block_sizes"]), int(header["bandwidth"]))
        except (KeyError, TypeError) as e:
            raise InvalidArgumentError(f"read_bbm: malformed header ({e})") from None
        m = BlockBandedMatrix(lay)
        payload = f.read()
    pos = 0
    for a, off in _inband(lay):
        r, c = lay.block_sizes[a], lay.block_sizes[a + off]
        nbytes = 16 * r * c
        if pos + nbytes > len(payload):
            raise InvalidArgumentError(f"read_bbm: truncated block data in {path}")
        blk = np.frombuffer(payload, dtype="<c16", count=r * c, offset=pos).reshape((r, c), order="F")
        m.data[a, off + lay.bandwidth, :r, :c] = blk
        pos += nbytes
    return m
