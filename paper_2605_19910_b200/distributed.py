"""Domain-sharded DDRGF across ranks: one process per GPU, torch.distributed (NCCL)
for the single interface exchange.

The decomposition is the reference's (interleave_permutation(layout, 1, s2),
partition.hpp:39-75): tasks t = [interior group t, separator t]. Ranks own
contiguous task ranges, hence contiguous layer ranges of the band. Protocol
(SURVEY.md 8(e)):

  1. phase 1 on every rank: fake-lead corners of its domains + interface A blocks
     -> one packet of 9 b x b blocks per task (csrc/ddrgf.cu);
  2. all-gather of the packets (the only data-path collective: 9 b^2 complex per
     task, e.g. 8 domains at b = 768: 680 MB over NVLink);
  3. phase 2, identical on every rank: left/right-connected sweeps over the P
     separators -> boundary self-energies, right-connected G, separator G;
  4. phase 3 on every rank: in-place RGF re-solve of its chains;
  5. all-gather of two boundary blocks per rank (the halo), then the couplings between
     chains, each consistent with the chain whose row of A G it closes.

The same protocol runs inside the library with NCCL (bbsi_cuda_ddrgf_rank_dev,
:func:`ddrgf_nccl`); this module keeps the phase-by-phase form for the CPU tests.

``engine`` is the phase implementation; production code always uses
:class:`CudaPhases` (the C ABI). The CPU tests inject a numpy restatement to run the
protocol under ``gloo`` with world size 2 (tests/test_distributed_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._native import lib
from .bbsi import _raise

PACKET_BLOCKS = 9
PHASE2_BLOCKS = 4


@dataclass(frozen=True)
class Task:
    first: int  # first interior layer (== sep when the group is empty)
    count: int  # interior layers
    sep: int    # separator layer


def partition(l: int, s2: int) -> list[Task]:
    """interleave_permutation(layout, 1, s2) groups (partition.hpp:39-75)."""
    out, pos = [], 0
    while pos < l:
        rem = l - pos
        if rem >= 1 + s2:
            d2, d1 = s2, 1
        else:
            d1 = min(1, rem)
            d2 = rem - d1
        out.append(Task(pos, d2, pos + d2))
        pos += d2 + d1
    return out


def task_ranges(n_tasks: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced task ranges per rank (at least one task per rank)."""
    if world > n_tasks:
        raise ValueError(f"{world} ranks for {n_tasks} DDRGF tasks")
    base, extra = divmod(n_tasks, world)
    out, t = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((t, t + n))
        t += n
    return out


def layer_range(tasks: list[Task], t0: int, t1: int) -> tuple[int, int]:
    """Band rows [L0, L1) owned by tasks t0..t1-1."""
    return tasks[t0].first, tasks[t1 - 1].sep + 1


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class CudaPhases:
    """The three DDRGF phases on the current CUDA device (C ABI, csrc/ddrgf.cu)."""

    def __init__(self, l: int, b: int, s2: int):
        self.l, self.b, self.s2 = l, b, s2
        self._G = None  # one band-sized work buffer: phase 1's scratch, then phase 3's result

    def _band(self, A_loc):
        import torch

        if self._G is None or self._G.shape != A_loc.shape or self._G.device != A_loc.device:
            self._G = torch.empty_like(A_loc)
        return self._G

    def phase1(self, A_loc, t0: int, t1: int):
        import torch

        G = self._band(A_loc)
        pk = torch.empty((t1 - t0, PACKET_BLOCKS, self.b, self.b), dtype=torch.complex128, device=A_loc.device)
        fail = C.c_int(-1)
        rc = lib().bbsi_cuda_ddrgf_phase1_dev(self.l, self.b, self.s2, t0, t1, _ptr(A_loc), _ptr(G), _ptr(pk),
                                              C.byref(fail), _stream())
        _raise(rc, fail.value)
        return pk

    def phase2(self, packets):
        import torch

        n = packets.shape[0]
        out = torch.empty((n, PHASE2_BLOCKS, self.b, self.b), dtype=torch.complex128, device=packets.device)
        fail = C.c_int(-1)
        rc = lib().bbsi_cuda_ddrgf_phase2_dev(self.l, self.b, self.s2, _ptr(packets), _ptr(out), C.byref(fail),
                                              _stream())
        _raise(rc, fail.value)
        return out

    def phase3(self, A_loc, out, t0: int, t1: int):
        G = self._band(A_loc)
        self._G = None  # handed to the caller
        fail = C.c_int(-1)
        rc = lib().bbsi_cuda_ddrgf_phase3_dev(self.l, self.b, self.s2, t0, t1, _ptr(A_loc), _ptr(G), _ptr(out),
                                              C.byref(fail), _stream())
        _raise(rc, fail.value)
        return G

    def halo(self, G, t0: int, t1: int):
        import torch

        h = torch.empty((2, self.b, self.b), dtype=torch.complex128, device=G.device)
        _raise(lib().bbsi_cuda_ddrgf_halo_dev(self.l, self.b, self.s2, t0, t1, _ptr(G), _ptr(h), _stream()))
        return h

    def couplings(self, A_loc, G, out, t0: int, t1: int, prev_sep_g=None, next_x0_g=None):
        p = _ptr(prev_sep_g) if prev_sep_g is not None else None
        n = _ptr(next_x0_g) if next_x0_g is not None else None
        _raise(lib().bbsi_cuda_ddrgf_couplings_dev(self.l, self.b, self.s2, t0, t1, _ptr(A_loc), _ptr(G), _ptr(out),
                                                   p, n, _stream()))
        return G


def gather_packets(packet, ranges, group=None):
    """All-gather of the per-rank packets into task order (padded to the largest range)."""
    import torch
    import torch.distributed as dist

    maxn = max(t1 - t0 for t0, t1 in ranges)
    pad = torch.zeros((maxn,) + tuple(packet.shape[1:]), dtype=packet.dtype, device=packet.device)
    pad[: packet.shape[0]] = packet
    world = len(ranges)
    # complex tensors travel as their real view (NCCL / gloo have no complex reduction needs here)
    flat = torch.view_as_real(pad).contiguous()
    bufs = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(bufs, flat, group=group)
    parts = [torch.view_as_complex(bufs[r])[: t1 - t0] for r, (t0, t1) in enumerate(ranges)]
    return torch.cat(parts, dim=0)


def ddrgf_distributed(A_loc, l: int, b: int, s2: int, group=None, engine=None):
    """Selected inverse rows [L0, L1) of this rank's task range (see layer_range).

    A_loc: complex128 (L1-L0, 3, b, b) band rows of this rank in slot order (column-major
    blocks, i.e. tensor[a, off+1, col, row]); returns G_loc of the same shape.
    """
    import torch.distributed as dist

    tasks = partition(l, s2)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ranges = task_ranges(len(tasks), world)
    t0, t1 = ranges[rank]
    eng = engine or CudaPhases(l, b, s2)
    packet = eng.phase1(A_loc, t0, t1)
    packets = gather_packets(packet, ranges, group) if world > 1 else packet
    out = eng.phase2(packets)
    G = eng.phase3(A_loc, out, t0, t1)
    halo = eng.halo(G, t0, t1)
    prev = nxt = None
    if world > 1:
        halos = gather_packets(halo[None], [(r, r + 1) for r in range(world)], group)  # [world][2]
        prev = halos[rank - 1, 1] if rank > 0 else None
        nxt = halos[rank + 1, 0] if rank + 1 < world else None
    return eng.couplings(A_loc, G, out, t0, t1, prev, nxt)


class NcclComm:
    """A NCCL communicator created by the library (one per rank); the unique id travels
    over torch.distributed (or any side channel) once."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _raise(lib().bbsi_cuda_nccl_unique_id(uid))
        if world > 1:
            dev = torch.device("cuda", torch.cuda.current_device())
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
            dist.broadcast(t, 0, group=group)
            uid = (C.c_ubyte * 128)(*t.cpu().tolist())
        self.comm = C.c_void_p()
        _raise(lib().bbsi_cuda_nccl_comm_init(uid, world, rank, C.byref(self.comm)))
        self.world, self.rank = world, rank

    def close(self):
        if self.comm:
            lib().bbsi_cuda_nccl_comm_destroy(self.comm)
            self.comm = C.c_void_p()


def rank_layers(l: int, s2: int, world: int, rank: int) -> tuple[int, int, int, int]:
    """(t0, t1, L0, L1): the task range and band rows a rank owns (C ABI)."""
    v = [C.c_int() for _ in range(4)]
    _raise(lib().bbsi_cuda_ddrgf_rank_layers(l, s2, world, rank, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def ddrgf_nccl(comm: NcclComm, A_loc, G_loc, l: int, b: int, s2: int, levels_above=()):
    """This rank's part of the domain-sharded DDRGF with NCCL inside the library
    (bbsi_cuda_ddrgf_rank_dev): A_loc / G_loc are the rank's band rows (rank_layers).
    levels_above: the DomainPlan's later levels s2_levels[1..] (ddrgf.hpp:363-369), which
    nest the interface system every rank solves (bbsi_cuda_ddrgf_rank_plan_dev)."""
    fail = C.c_int(-1)
    if levels_above:
        import numpy as np

        lv = np.array([s2, *levels_above], dtype=np.int32)
        rc = lib().bbsi_cuda_ddrgf_rank_plan_dev(comm.comm, l, b, lv.ctypes.data_as(C.c_void_p), len(lv),
                                                 _ptr(A_loc), _ptr(G_loc), C.byref(fail), _stream())
    else:
        rc = lib().bbsi_cuda_ddrgf_rank_dev(comm.comm, l, b, s2, _ptr(A_loc), _ptr(G_loc), C.byref(fail), _stream())
    _raise(rc, fail.value)
    return G_loc
