"""CSMR tensor files, dataset directories and the CLI (the reference's
test_io.py / test_cli.py behaviours).  File handling
and argument checking run on CPU; the reconstructions are -m gpu."""

import json
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_2006_14080_b200 import cli
from paper_2006_14080_b200.acquisition import Trajectory
from paper_2006_14080_b200.io import (TensorFileError, load_dataset, read_tensor,
                                      save_dataset, write_tensor)

DTYPES = [np.complex64, np.complex128, np.float32, np.float64]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", [(7,), (3, 5), (2, 3, 4), (1, 1, 1, 2)])
def test_bitwise_round_trip(tmp_path, dtype, shape):
    rng = np.random.default_rng(3)
    a = rng.standard_normal(shape)
    if np.issubdtype(dtype, np.complexfloating):
        a = a + 1j * rng.standard_normal(shape)
    a = a.astype(dtype)
    a.flat[0] = np.nan if a.size > 1 else a.flat[0]  # NaN payload survives too
    write_tensor(tmp_path / "t.cplx", a)
    b = read_tensor(tmp_path / "t.cplx")
    assert b.dtype == np.dtype(dtype).newbyteorder("<") and b.shape == a.shape
    assert a.tobytes() == b.tobytes()


def test_non_contiguous_and_fortran_inputs(tmp_path):
    a = (np.arange(24.0).reshape(4, 6) + 1j).astype(np.complex64)
    for v in (a[:, ::2], np.asfortranarray(a)):
        write_tensor(tmp_path / "v.cplx", v)
        assert np.array_equal(read_tensor(tmp_path / "v.cplx"), v)


def test_exact_byte_layout(tmp_path):
    a = np.array([[1 + 2j, 3 - 4j]], dtype=np.complex64)
    write_tensor(tmp_path / "x.cplx", a)
    raw = (tmp_path / "x.cplx").read_bytes()
    assert raw[:8] == b"CSMR" + bytes([1, 0, 2, 0])
    assert struct.unpack("<2Q", raw[8:24]) == (1, 2)
    assert np.frombuffer(raw[24:], "<f4").tolist() == [1, 2, 3, -4]


def test_dtype_codes(tmp_path):
    for code, dt in enumerate(DTYPES):
        write_tensor(tmp_path / "c.cplx", np.zeros(2, dt))
        assert (tmp_path / "c.cplx").read_bytes()[5] == code


def _corrupt(tmp_path, mutate):
    write_tensor(tmp_path / "g.cplx", np.ones((2, 3), np.complex64))
    raw = bytearray((tmp_path / "g.cplx").read_bytes())
    raw = mutate(raw)
    (tmp_path / "g.cplx").write_bytes(bytes(raw))
    return tmp_path / "g.cplx"


@pytest.mark.parametrize("mutate,match", [
    (lambda r: b"XSMR" + r[4:], "magic"),
    (lambda r: r[:4] + bytes([2]) + r[5:], "version"),
    (lambda r: r[:5] + bytes([9]) + r[6:], "dtype code"),
    (lambda r: r[:6] + bytes([0]) + r[7:], "ndim"),
    (lambda r: r[:5], "truncated header"),
    (lambda r: r[:12], "dimension list"),
    (lambda r: r[:-1], "payload"),
    (lambda r: r + b"\0", "payload"),
])
def test_malformed_files_rejected(tmp_path, mutate, match):
    with pytest.raises(TensorFileError, match=match):
        read_tensor(_corrupt(tmp_path, mutate))


def test_unsupported_arrays_rejected_on_write(tmp_path):
    with pytest.raises(TensorFileError, match="unsupported dtype"):
        write_tensor(tmp_path / "i.cplx", np.arange(3))
    with pytest.raises(TensorFileError, match="ndim"):
        write_tensor(tmp_path / "z.cplx", np.float64(1.0))


def _small_dataset(tmp_path, name="ds"):
    from harness.configs import make_problem
    prob = make_problem(0)
    traj = Trajectory(prob.coords, 32, 128)
    meta = {"config": 0, "seed": "harness"}
    save_dataset(tmp_path / name, prob.truth, prob.sens, traj, prob.data, meta)
    return tmp_path / name, prob


def test_dataset_round_trip_and_derived_meta(tmp_path):
    d, prob = _small_dataset(tmp_path)
    phantom, sens, ds, meta = load_dataset(d)
    assert np.array_equal(phantom, prob.truth.astype(np.complex128))
    assert np.array_equal(sens.maps, prob.sens) and np.array_equal(ds.data, prob.data)
    assert np.array_equal(ds.trajectory.coords, prob.coords)
    assert meta["n_readouts_kept"] == 32 and meta["n_samples_per_readout"] == 128
    assert meta["n_kspace_samples"] == 4096 and meta["n_coils"] == 4
    json.loads((d / "meta.json").read_text())


def test_saves_are_byte_identical(tmp_path):
    a, _ = _small_dataset(tmp_path, "a")
    b, _ = _small_dataset(tmp_path, "b")
    for f in ("phantom.cplx", "sens.cplx", "traj.cplx", "kspace.cplx", "meta.json"):
        assert (a / f).read_bytes() == (b / f).read_bytes()


def test_missing_meta_rejected(tmp_path):
    (tmp_path / "empty").mkdir()
    with pytest.raises(TensorFileError, match="meta.json"):
        load_dataset(tmp_path / "empty")


def _run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2006_14080_b200", *args],
                          capture_output=True, text=True)


def test_usage_errors_exit_2(tmp_path):
    assert _run_cli("reconstruct", "--data", str(tmp_path)).returncode == 2
    assert _run_cli("reconstruct", "--data", str(tmp_path), "--out", "x",
                    "--workers", "0").returncode == 2
    assert _run_cli("benchmark", "--data", str(tmp_path), "--out", "x.csv",
                    "--workers-list", ",").returncode == 2


def test_runtime_errors_exit_1(tmp_path, capsys):
    assert cli.main(["reconstruct", "--data", str(tmp_path / "missing"),
                     "--out", str(tmp_path / "img.cplx")]) == 1
    assert "error:" in capsys.readouterr().err
    d, _ = _small_dataset(tmp_path)
    # double precision has no GPU path and no CPU fallback
    assert cli.main(["reconstruct", "--data", str(d), "--out", str(tmp_path / "i.cplx"),
                     "--precision", "f64"]) == 1


@pytest.mark.gpu
def test_cli_adjoint_matches_library(tmp_path):
    import paper_2006_14080_b200 as P
    d, _ = _small_dataset(tmp_path)
    out = tmp_path / "adj.cplx"
    assert cli.main(["reconstruct", "--data", str(d), "--out", str(out),
                     "--method", "adjoint"]) == 0
    _, sens, ds, _ = load_dataset(d)
    ref, _ = P.adjoint_reconstruct(ds, sens)
    assert np.array_equal(read_tensor(out), np.asarray(ref))


@pytest.mark.gpu
def test_cli_admm_writes_image_report_and_is_repeatable(tmp_path):
    d, _ = _small_dataset(tmp_path)
    outs = []
    for k in range(2):
        out = tmp_path / f"img{k}.cplx"
        assert cli.main(["reconstruct", "--data", str(d), "--out", str(out),
                         "--admm-iters", "3", "--cg-iters", "5"]) == 0
        rep = json.loads((tmp_path / f"img{k}.cplx.report.json").read_text())
        assert rep["method"] == "admm" and len(rep["iterations"]) <= 3
        assert rep["dataset"] == str(d) and rep["image"] == str(out)
        outs.append(out.read_bytes())
    assert outs[0] == outs[1]  # deterministic device reductions


@pytest.mark.gpu
def test_cli_benchmark_single_worker_row(tmp_path):
    d, _ = _small_dataset(tmp_path)
    out = tmp_path / "bench.csv"
    assert cli.main(["benchmark", "--data", str(d), "--out", str(out),
                     "--workers-list", "1", "--repeat", "1", "--admm-iters", "2"]) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "workers,best_seconds,speedup,ideal_speedup,note"
    assert rows[1].startswith("1,") and ",1.000,1.000," in rows[1]


def test_shard_flag_is_validated():
    assert _run_cli("reconstruct", "--data", "d", "--out", "x", "--shard",
                    "tiles").returncode == 2


@pytest.mark.gpu
def test_cli_sample_shard_matches_library(tmp_path):
    # --shard sample: the order-stable plan through the CLI == the library call
    import paper_2006_14080_b200 as P
    d, _ = _small_dataset(tmp_path)
    out = tmp_path / "img_s.cplx"
    assert cli.main(["reconstruct", "--data", str(d), "--out", str(out), "--admm-iters", "3",
                     "--cg-iters", "5", "--shard", "sample"]) == 0
    rep = json.loads((tmp_path / "img_s.cplx.report.json").read_text())
    assert rep["timing"]["shard"] == "sample"
    _, sens, ds, _ = load_dataset(d)
    params = P.ReconParams(lam=1e-7, beta=1.0, admm_rtol=1e-4, admm_max_iters=3,
                           cg_atol=1e-6, cg_max_iters=5)
    ref, _ = P.admm_reconstruct(ds, sens, params, shard="sample", compute_objectives=False)
    assert np.array_equal(read_tensor(out), np.asarray(ref))
