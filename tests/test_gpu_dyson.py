"""Parity of the resident Dyson batch path (BASELINE configs) against the oracle.

Bar (BASELINE.json north_star): per-block relative Frobenius error <= 1e-10 of
every diagonal and off-diagonal G^R block against the reference CPU RGF on the
same seeded input. Config 1 runs at full size (also against the dense oracle);
configs 2/3 at reduced layer / energy counts with their true b, w and eta
(full-size checks live in tests/test_gpu_dyson_full.py).
"""
import numpy as np
import pytest

from oracle import bbsi_oracle as O
from oracle import dyson_oracle as DO
from paper_2605_19910_b200 import dyson as D

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _run_gpu(cfg):
    import torch

    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((cfg.n_energy, l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    fails = D.solve_device(cfg, H, G)
    assert (fails == -1).all()
    torch.cuda.synchronize()
    return np.swapaxes(G.cpu().numpy(), -1, -2)  # slot memory -> (row, col)


def _oracle_band(cfg, e):
    h = DO.hamiltonian(cfg.num_layers, cfg.bandwidth, cfg.block_size, cfg.seed)
    return DO.dyson_matrix(h, complex(cfg.z()[e]), cfg.sigma_layers)


def _check(cfg, dense=False, energies=None):
    g = _run_gpu(cfg)
    lay = O.make_layout(cfg.num_layers, cfg.block_size, cfg.bandwidth)
    worst = 0.0
    for e in energies if energies is not None else range(cfg.n_energy):
        a = _oracle_band(cfg, e)
        ref = O.rgf_ndiag(a)[0] if cfg.bandwidth > 1 else O.rgf_tridiag(a)[0]
        got = O.Band(lay, g[e])
        err = O.max_block_error(got, ref)
        worst = max(worst, err)
        assert err <= TOL, (e, err)
        if dense:
            assert O.max_block_error(got, O.oracle_selected_inverse(a)) <= TOL
    return worst


def test_config1_full_size_vs_rgf_and_dense(gpu):
    _check(D.CONFIGS[1], dense=True)


def test_config2_proxy(gpu):
    _check(D.scaled(D.CONFIGS[2], num_layers=24, n_energy=4))


def test_config3_proxy(gpu):
    _check(D.scaled(D.CONFIGS[3], num_layers=24, n_energy=4))


def test_config5_block_size_proxy(gpu):
    _check(D.scaled(D.CONFIGS[5], num_layers=6, n_energy=2))


@pytest.mark.parametrize("cfg_id,layers,n_e,b,chunk", [(2, 20, 10, 64, 0), (2, 20, 10, 64, 3), (3, 11, 3, 64, 0)])
def test_host_path_streams_identical_bands(gpu, cfg_id, layers, n_e, b, chunk):
    """bbsi_cuda_dyson_rgf_z (host buffers, rows streamed during the downward sweep,
    optional energy chunks) returns exactly the resident path's bands."""
    cfg = D.scaled(D.CONFIGS[cfg_id], num_layers=layers, n_energy=n_e, block_size=b)
    dev = np.swapaxes(_run_gpu(cfg), -1, -2)  # back to slot memory
    got, fails = D.solve_host(cfg, chunk=chunk)
    assert (fails == -1).all()
    assert np.array_equal(got, dev)
    lay = O.make_layout(cfg.num_layers, cfg.block_size, cfg.bandwidth)
    for e in (0, n_e - 1):
        a = _oracle_band(cfg, e)
        ref = O.rgf_ndiag(a)[0] if cfg.bandwidth > 1 else O.rgf_tridiag(a)[0]
        assert O.max_block_error(O.Band(lay, np.swapaxes(got[e], -1, -2)), ref) <= TOL


@pytest.mark.parametrize("layers,n_e", [(3, 2), (4, 3), (5, 9), (8, 9), (33, 4)])
def test_two_ended_sweep_layer_counts(gpu, layers, n_e):
    """The Dyson batch runs the two-ended tridiagonal sweep (chains meet at l/2):
    odd / even / minimal layer counts, one and two stream groups, against the
    reference's one-ended RGF."""
    _check(D.scaled(D.CONFIGS[2], num_layers=layers, n_energy=n_e, block_size=64))


_BANDED_CASES = [(2, 8, 2), (2, 9, 3), (2, 10, 9), (2, 7, 2), (3, 11, 2), (3, 16, 3), (2, 24, 4)]


def _in_subprocess(env, code):
    """Runs `code` in a fresh interpreter (the library reads its switches once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_one_ended_banded_sweep(gpu):
    """The one-ended banded recursion (BBSI_TWO_ENDED_BANDED=0; the default is two-ended:
    chains from both ends, the w middle layers inverted as one dense (w b)^2 matrix,
    outward sweeps; one-ended below l = 3w + 2) against the reference's rgf_ndiag, and the
    host path's streamed rows against the resident bands."""
    code = f"""
import numpy as np
from dataclasses import replace
import tests.test_gpu_dyson as T
from paper_2605_19910_b200 import dyson as D
for w, layers, n_e in {_BANDED_CASES}:
    T._check(replace(D.scaled(D.CONFIGS[3], num_layers=layers, n_energy=n_e, block_size=64), bandwidth=w))
for w, layers in ((2, 14), (3, 20)):
    cfg = replace(D.scaled(D.CONFIGS[3], num_layers=layers, n_energy=3, block_size=64), bandwidth=w)
    dev = np.swapaxes(T._run_gpu(cfg), -1, -2)
    got, fails = D.solve_host(cfg)
    assert (fails == -1).all() and np.array_equal(got, dev)
print("ok")
"""
    _in_subprocess({"BBSI_TWO_ENDED_BANDED": "0"}, code)


def test_switches_keep_results(gpu, tmp_path):
    """The Dyson diagonal blocks formed inside the first Schur-update GEMM give bit-identical
    bands to the separate forming pass (BBSI_FORM_IN_GEMM=0), and the one-ended sweep
    (BBSI_TWO_ENDED=0) agrees with the default two-ended one to rounding."""
    out = {}
    for tag, env in (("default", {}), ("form_pass", {"BBSI_FORM_IN_GEMM": "0"}), ("one_ended", {"BBSI_TWO_ENDED": "0"})):
        f = tmp_path / f"{tag}.npy"
        code = f"""
import numpy as np
import tests.test_gpu_dyson as T
from paper_2605_19910_b200 import dyson as D
cfg = D.scaled(D.CONFIGS[2], num_layers=21, n_energy=10, block_size=64)
np.save({str(f)!r}, T._run_gpu(cfg))
"""
        _in_subprocess(env, code)
        out[tag] = np.load(f)
    assert np.array_equal(out["default"], out["form_pass"])
    ref = out["one_ended"]
    nrm = np.linalg.norm(ref, axis=(-2, -1))
    err = np.linalg.norm(out["default"] - ref, axis=(-2, -1))
    assert (err <= 1e-10 * np.maximum(nrm, 1e-300)).all(), float((err / np.maximum(nrm, 1e-300)).max())


def test_host_path_graph_replay_pinned(gpu):
    """With pinned host buffers the host path is captured once and replayed as a CUDA
    graph (H2D, sweeps, the streamed D2H of G): replays give the resident bands, also
    after H and z change between calls."""
    import torch

    cfg = D.scaled(D.CONFIGS[2], num_layers=20, n_energy=50, block_size=64)  # three chunks
    dev = np.swapaxes(_run_gpu(cfg), -1, -2)
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    Hh = torch.from_numpy(D.fill_h_host(cfg)).pin_memory()
    Gh = torch.empty((cfg.n_energy, l, 2 * w + 1, b, b), dtype=torch.complex128).pin_memory()
    z = np.ascontiguousarray(cfg.z())
    for _ in range(3):  # eager, capture, replay
        Gh.zero_()
        got, fails = D.solve_host(cfg, H=Hh.numpy(), z=z, G=Gh.numpy())
        assert (fails == -1).all()
        assert np.array_equal(got, dev)
    # same buffers, new contents: the replay reads them again
    z2 = z + 0.01
    Gh.zero_()
    got2, _ = D.solve_host(cfg, H=Hh.numpy(), z=z2, G=Gh.numpy())
    ref2, _ = D.solve_host(cfg, H=np.array(Hh.numpy()), z=z2)  # pageable: eager path
    assert np.array_equal(got2, ref2)


def test_full_sigma_blocks(gpu):
    """Dyson batch with full, energy-dependent lead self-energy blocks on the first and last
    w layers (bbsi_cuda_dyson_rgf_sigma_dev) against the oracle RGF of the same A(E)."""
    import torch
    from dataclasses import replace

    for w, l, b in ((1, 12, 64), (2, 14, 64)):
        cfg = replace(D.scaled(D.CONFIGS[3 if w == 2 else 2], num_layers=l, n_energy=3, block_size=b), bandwidth=w)
        rng = np.random.default_rng(5)
        ne = cfg.n_energy
        sig = (rng.uniform(-0.3, 0.3, (ne, 2 * w, b, b)) + 1j * rng.uniform(-0.6, 0.0, (ne, 2 * w, b, b)))
        H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
        D.fill_h_device(cfg, H)
        G = torch.empty((ne, l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
        dsig = torch.from_numpy(np.ascontiguousarray(np.swapaxes(sig, -1, -2))).cuda()  # slot (column-major) blocks
        D.solve_device_sigma(cfg, H, G, dsig)
        torch.cuda.synchronize()
        h = DO.hamiltonian(l, w, b, cfg.seed)
        for e, z in enumerate(cfg.z()):
            a = DO.dyson_matrix(h, complex(z), 0)
            for q in range(2 * w):
                layer = q if q < w else l - 2 * w + q
                a.block(layer, 0)[...] -= sig[e, q]
            ref, _ = (O.rgf_ndiag if w > 1 else O.rgf_tridiag)(a)
            got = O.Band(ref.layout, np.swapaxes(G[e].cpu().numpy(), -1, -2))
            assert O.max_block_error(got, ref) <= 1e-10
