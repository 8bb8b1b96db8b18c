"""Multi-rank DDRGF protocol on CPU: world size 2 over gloo, numpy phase engine
(tests/_ddrgf_np_engine.py) behind paper_2605_19910_b200.distributed, compared with
the sequential RGF oracle. Also checks the task partition against the reference."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bbsi_oracle as O
from oracle import dyson_oracle as DO
from paper_2605_19910_b200 import distributed as Dd

CASES = [(23, 16, 4), (30, 16, 5), (20, 32, 3), (17, 16, 7)]  # (l, b, s2), incl. trailing groups


def _matrix(l, b):
    return DO.dyson_matrix(DO.hamiltonian(l, 1, b, 9), complex(0.15, 1e-4), 1)


def _slots(m: O.Band):
    return torch.from_numpy(np.ascontiguousarray(m.data.transpose(0, 1, 3, 2)))


def test_partition_matches_reference():
    for l, s2 in ((10, 4), (11, 4), (12, 4), (2, 1), (4096, 511), (2048, 255)):
        _, desc = O.interleave_permutation(O.make_layout(l, 1, 1), 1, s2)
        tasks = Dd.partition(l, s2)
        assert [(t.first, t.count) for t in tasks] == [tuple(g) for g in desc.interior_groups]
        assert [t.sep for t in tasks] == [g[0] for g in desc.separator_groups]


def test_task_ranges_cover_and_balance():
    for n, w in ((8, 2), (8, 8), (9, 4), (33, 8)):
        r = Dd.task_ranges(n, w)
        assert r[0][0] == 0 and r[-1][1] == n and all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("l,b,s2", CASES)
def test_single_rank_protocol_numpy_engine(l, b, s2):
    from tests._ddrgf_np_engine import NumpyPhases

    a = _matrix(l, b)
    G = Dd.ddrgf_distributed(_slots(a), l, b, s2, engine=NumpyPhases(l, b, s2))
    got = O.Band(a.layout, np.ascontiguousarray(G.numpy().transpose(0, 1, 3, 2)))
    assert O.max_block_error(got, O.rgf_tridiag(a)[0]) <= 1e-10


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        from tests._ddrgf_np_engine import NumpyPhases

        l, b, s2 = case
        a = _matrix(l, b)
        tasks = Dd.partition(l, s2)
        t0, t1 = Dd.task_ranges(len(tasks), world)[rank]
        L0, L1 = Dd.layer_range(tasks, t0, t1)
        A_loc = _slots(a)[L0:L1].clone()
        G_loc = Dd.ddrgf_distributed(A_loc, l, b, s2, engine=NumpyPhases(l, b, s2))
        parts = [None] * world
        dist.all_gather_object(parts, (L0, L1, G_loc.numpy()))
        if rank == 0:
            full = np.zeros((l, 3, b, b), dtype=np.complex128)
            for lo, hi, g in parts:
                full[lo:hi] = g
            got = O.Band(a.layout, np.ascontiguousarray(full.transpose(0, 1, 3, 2)))
            q.put(O.max_block_error(got, O.rgf_tridiag(a)[0]))
        del sys
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES[:2])
def test_two_ranks_gloo(case):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert err <= 1e-10


def test_rank_layers_c_abi_matches_protocol():
    """bbsi_cuda_ddrgf_rank_layers (host-only C ABI, used by the NCCL path inside the
    library) agrees with the Python protocol's task ranges and band rows."""
    for l, s2, world in ((4096, 127, 8), (4096, 511, 8), (2048, 255, 4), (30, 5, 3), (17, 7, 2), (23, 4, 5)):
        tasks = Dd.partition(l, s2)
        for rank, (t0, t1) in enumerate(Dd.task_ranges(len(tasks), world)):
            L0, L1 = Dd.layer_range(tasks, t0, t1)
            assert Dd.rank_layers(l, s2, world, rank) == (t0, t1, L0, L1)
    from paper_2605_19910_b200 import InvalidArgumentError

    with pytest.raises(InvalidArgumentError):
        Dd.rank_layers(30, 5, 6, 0)  # 5 domains, 6 ranks
