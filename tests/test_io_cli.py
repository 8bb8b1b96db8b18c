""".bbm I/O (io.cpp:26-75), the product-side random_spd_like generator and the `bbsi`
CLI (tools/bbsi.cpp) -- CPU checks against the reference's own files and generator,
plus GPU runs of the CLI's solve / validate paths."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2605_19910_b200 as P
from oracle import bbsi_oracle as O
from paper_2605_19910_b200 import cli

GOLDEN = Path(__file__).resolve().parent / "golden"


def _fixture_l5():
    m = P.random_spd_like(P.make_layout(5, 3, 2), 99, 2.0)
    m.data[0, 2, 0, 0] = complex(-0.0, 1e-308)  # test_io.cpp:24-26
    return m


@pytest.mark.parametrize("layout", [((5, 3, 2), None), ((4, None, 1), [2, 5, 1, 3]), ((1, 4, 0), None),
                                    ((9, 2, 3), None)])
def test_generator_bit_exact_vs_oracle(layout):
    (l, b, w), sizes = layout
    lay = P.make_layout(l, b, w) if sizes is None else P.BlockLayout(l, sizes, w)
    olay = O.make_layout(l, b, w) if sizes is None else O.BlockLayout(l, sizes, w)
    assert np.array_equal(P.random_spd_like(lay, 4242, 1.5).data, O.random_spd_like(olay, 4242, 1.5).data)


def test_generator_rejects_bad_dominance():
    with pytest.raises(P.InvalidArgumentError):
        P.random_spd_like(P.make_layout(3, 2, 1), 1, 0.0)


def test_read_reference_written_files():
    """Files written by the reference's write_bbm (tests/golden/make_golden.py) read back
    bit-exactly, signed zero and subnormal included (test_io.cpp:22-38)."""
    m = P.read_bbm(str(GOLDEN / "io_l5_b3_w2_s99.bbm"))
    ref = _fixture_l5()
    assert m.layout == ref.layout
    assert np.array_equal(m.data.view(np.uint64), ref.data.view(np.uint64))
    assert np.signbit(m.block(0, 0)[0, 0].real)
    r = P.read_bbm(str(GOLDEN / "io_ragged_l4_s123.bbm"))
    assert r.layout.block_sizes == [2, 5, 1, 3]
    assert np.array_equal(r.data, P.random_spd_like(P.BlockLayout(4, [2, 5, 1, 3], 1), 123, 2.0).data)


@pytest.mark.parametrize("name,make", [("io_l5_b3_w2_s99.bbm", _fixture_l5),
                                       ("io_ragged_l4_s123.bbm",
                                        lambda: P.random_spd_like(P.BlockLayout(4, [2, 5, 1, 3], 1), 123, 2.0))])
def test_written_bytes_identical_to_reference(tmp_path, name, make):
    out = tmp_path / name
    P.write_bbm(str(out), make())
    assert out.read_bytes() == (GOLDEN / name).read_bytes()


def test_reference_reads_our_files(tmp_path):
    from oracle import ref_lib as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    m = P.random_spd_like(P.BlockLayout(6, [3, 1, 4, 2, 3, 2], 2), 7, 2.0)
    P.write_bbm(str(tmp_path / "x.bbm"), m)
    back = R.read_bbm(tmp_path / "x.bbm")
    assert np.array_equal(back.data, m.data)


def test_read_rejections(tmp_path):
    """test_io.cpp:40-66 plus the header checks of io.cpp:52-57."""
    with pytest.raises(P.InvalidArgumentError):
        P.read_bbm("/tmp/bbsi_test_definitely_absent.bbm")
    junk = tmp_path / "junk.bbm"
    junk.write_text("not a header\n")
    with pytest.raises(P.InvalidArgumentError, match="malformed"):
        P.read_bbm(str(junk))
    good = (GOLDEN / "io_l5_b3_w2_s99.bbm").read_bytes()
    trunc = tmp_path / "trunc.bbm"
    trunc.write_bytes(good[:-16])
    with pytest.raises(P.InvalidArgumentError, match="truncated"):
        P.read_bbm(str(trunc))
    hdr, body = good.split(b"\n", 1)
    for key, val, msg in (("version", 2, "version"), ("scalar", "c64", "scalar")):
        h = json.loads(hdr)
        h[key] = val
        f = tmp_path / f"bad_{key}.bbm"
        f.write_bytes(json.dumps(h).encode() + b"\n" + body)
        with pytest.raises(P.InvalidArgumentError, match=msg):
            P.read_bbm(str(f))


def test_cli_plan_parsing_and_dense_check():
    o = cli.argparse.Namespace(plan="s2:4,1,1", threads=3, terminal_threads=2)
    p = cli.parse_plan(o)
    assert p.s2_levels == [4, 1, 1] and p.n_threads == 3 and p.terminal_threads == 2
    assert cli.parse_plan(cli.argparse.Namespace(plan="", threads=1, terminal_threads=1)).s2_levels == [1]
    # the CLI's dense check on the oracle's exact selected inverse
    m = P.random_spd_like(P.make_layout(6, 3, 1), 5, 2.0)
    om = O.Band(O.make_layout(6, 3, 1), m.data.copy())
    g = P.BlockBandedMatrix(m.layout, O.rgf_tridiag(om)[0].data)
    err, _ = cli.oracle_error(g, m)
    assert err < 1e-13
    g.data[2, 1, 0, 0] += 1.0
    err, where = cli.oracle_error(g, m)
    assert err > 1e-3 and where == (2, 2)


def test_cli_without_gpu_fails_loudly(capsys):
    from paper_2605_19910_b200._native import lib

    if lib().bbsi_cuda_device_count() > 0:
        pytest.skip("GPU present")
    rc = cli.main(["solve", "--layers", "4", "--block-size", "2", "--reps", "1"])
    assert rc == 2
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("solver,extra", [("rgf", []), ("nrgf", ["--bandwidth", "2"]), ("fused", ["--bandwidth", "2"]),
                                          ("ddrgf", ["--plan", "s2:3"])])
def test_cli_validate_on_gpu(gpu, tmp_path, capsys, solver, extra):
    rc = cli.main(["validate", "--solver", solver, "--layers", "13", "--block-size", "5", "--reps", "2",
                   "--seed", "9", *extra])
    rec = json.loads(capsys.readouterr().out)
    assert rc == 0
    assert rec["max_block_error"] <= 1e-10
    assert rec["repetitions"] == 2 and rec["solver"] == solver


@pytest.mark.gpu
def test_cli_matrix_file_and_scale(gpu, tmp_path, capsys):
    m = P.random_spd_like(P.BlockLayout(6, [3, 1, 4, 2, 3, 2], 1), 11, 2.0)
    P.write_bbm(str(tmp_path / "m.bbm"), m)
    out = tmp_path / "rec.json"
    rc = cli.main(["validate", "--matrix", str(tmp_path / "m.bbm"), "--reps", "1", "--out", str(out)])
    assert rc == 0 and json.loads(out.read_text())["max_block_error"] <= 1e-10
    rc = cli.main(["scale", "--axis", "layers", "--grid", "8,16", "--block-size", "4", "--reps", "1"])
    lines = capsys.readouterr().out.strip().splitlines()
    assert rc == 0 and lines[0].startswith("axis,value") and lines[-1].startswith("# loglog_slope")
    assert cli.main(["validate", "--layers", "90", "--block-size", "64", "--reps", "1"]) == 2  # above --oracle-cap


def test_cli_tune_from_ratios_file(tmp_path, capsys):
    """`tune --ratios-file` needs no GPU: the reference autotune on given ratios
    (tools/bbsi.cpp:318-350 record layout)."""
    f = tmp_path / "r.json"
    f.write_text(json.dumps({"block_size": 64, "t_gemm_us": 10.0, "r_lu": 2.0, "r_getrs": 1.0, "samples": 5}))
    rc = cli.main(["tune", "--ratios-file", str(f), "--layers", "512", "--threads", "64"])
    rec = json.loads(capsys.readouterr().out)
    assert rc == 0 and rec["choice"] == "ddrgf" and rec["plan"][-1]["terminal"]
    assert rec["ratios"]["t_gemm_us"] == 10.0


@pytest.mark.gpu
def test_cli_bench_kernels_and_tune_on_gpu(gpu, capsys):
    assert cli.main(["bench-kernels", "--sizes", "64,100", "--samples", "2", "--batch", "4"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "block_size,t_gemm_us,r_lu,r_getrs,samples" and len(lines) == 3
    assert float(lines[1].split(",")[1]) > 0
    rc = cli.main(["tune", "--layers", "64", "--block-size", "64", "--samples", "2", "--execute", "--reps", "1",
                   "--threads", "4"])
    rec = json.loads(capsys.readouterr().out)
    assert rc == 0 and "gpu_plan" in rec and rec["measured_rgf_ms"] > 0
