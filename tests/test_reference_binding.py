"""The reference's own code running on the B200 kernels (drop-in proof).

``paper_2006_14080_b200.refbind.install`` puts a ``"cuda"`` entry into the
reference's kernel table (kernels.py:212-231) and makes it active; the
reference's unmodified DftOperator, transform functions, admm_reconstruct
and adjoint_reconstruct (staged in oracle/_ref by oracle/build_ref.py) then
run every NUDFT, finite difference and soft threshold through the C ABI.
Results are held to the golden fixtures the reference produced in f64.
Also covers the one-shot C entries with the reference's kernel signatures
(csr_nudft_forward_sep / csr_nudft_adjoint_sep).
"""

import ctypes

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import csrecon_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(cuda):
    from oracle import build_ref
    if not build_ref.available():
        pytest.skip("oracle/_ref not staged (run oracle/build_ref.py where /root/reference exists)")
    cs = build_ref.load()
    import paper_2006_14080_b200.refbind as rb
    prev = rb.install(cs.kernels)
    yield cs
    rb.uninstall(cs.kernels, prev)


def test_table_is_active(ref):
    assert ref.kernels.active_backend() == "cuda"
    assert set(ref.kernels.get_impl("cuda")) >= {"forward_sep", "adjoint_sep", "theta",
                                                 "theta_adj", "soft"}


def test_reference_operator_on_b200(ref):
    from csrecon.acquisition import ImageGrid, SensitivityMaps
    from csrecon.operators import DftOperator
    g = golden("operators.npz")
    worst = 0.0
    for i in range(int(g["n_cases"])):
        p = f"c{i}_"
        nx, ny = g[p + "image"].shape
        op = DftOperator.build(g[p + "coords"], ImageGrid(nx, ny), SensitivityMaps(g[p + "sens"]),
                               mode="separable", precision="single")
        fwd = op.forward(g[p + "image"].astype(np.complex64))
        adj = op.adjoint(g[p + "y"].astype(np.complex64))
        assert fwd.dtype == np.complex64 and adj.dtype == np.complex64
        ef, ea = rel_err(fwd, g[p + "fwd_double"]), rel_err(adj, g[p + "adj_double"])
        worst = max(worst, ef, ea)
        assert ef <= 1e-5 and ea <= 1e-5, (i, ef, ea)
    print("reference DftOperator on the B200 kernels: worst rel-L2", worst)


def test_reference_transform_on_b200(ref):
    from csrecon.transform import soft_threshold, theta, theta_adjoint
    g = golden("transform.npz")
    assert np.array_equal(theta(g["img"].astype(np.complex64)), g["theta_single"])
    assert np.array_equal(theta_adjoint(g["stack"].astype(np.complex64)), g["theta_adj_single"])
    out = soft_threshold(g["z"].astype(np.complex64), float(g["t"]))
    assert np.array_equal(out == 0, g["soft_single"] == 0)


def test_reference_admm_on_b200(ref):
    from csrecon.acquisition import KSpaceDataset, SensitivityMaps, Trajectory
    from csrecon.solver import ReconParams, admm_reconstruct, adjoint_reconstruct
    g = golden("admm_small.npz")
    # Python floats, as the fixture's own run used (numpy float64 parameters
    # would promote the reference's single-precision vectors to complex128)
    lam, beta, rtol, na, atol, ncg = (float(v) for v in g["fixed_params"])
    params = ReconParams(lam=lam, beta=beta, admm_rtol=rtol, admm_max_iters=int(na),
                         cg_atol=atol, cg_max_iters=int(ncg))
    ds = KSpaceDataset(g["data"], Trajectory(g["coords"], g["coords"].shape[0], 1))
    sens = SensitivityMaps(g["sens"])
    for workers, order_stable in ((1, True), (2, True), (2, False)):
        img, rep = admm_reconstruct(ds, sens, params, n_workers=workers, precision="single",
                                    op_mode="separable", order_stable=order_stable)
        err = rel_err(img, g["fixed_double_image"])
        print(f"reference admm_reconstruct on the B200 kernels, {workers} workers, "
              f"order_stable={order_stable}: rel-L2 {err:.2e}")
        assert rep.backend == "cuda"
        assert err <= 1e-4
        obj = [rep.objective_initial] + [r["objective"] for r in rep.iterations]
        np.testing.assert_allclose(obj, g["fixed_double_obj"], rtol=1e-4)
    adj, _ = adjoint_reconstruct(ds, sens, precision="single", op_mode="separable")
    assert rel_err(adj, g["adjoint_double"]) <= 1e-5


def test_materialized_mode_is_refused(ref):
    from csrecon.acquisition import ImageGrid, SensitivityMaps
    from csrecon.operators import DftOperator
    g = golden("operators.npz")
    op = DftOperator.build(g["c1_coords"], ImageGrid(*g["c1_image"].shape),
                           SensitivityMaps(g["c1_sens"]), mode="materialized",
                           precision="single")
    with pytest.raises(NotImplementedError):
        op.forward(g["c1_image"].astype(np.complex64))


def test_oneshot_entries_with_reference_signatures(cuda):
    # kernels.nudft_forward_sep(phase0, phase1_t, sens, image) and
    # nudft_adjoint_sep(phase0, phase1_conj, sens, data) (kernels.py:257-262)
    import torch
    from paper_2006_14080_b200 import _native
    g = golden("operators.npz")
    lib = _native.load()
    st = torch.cuda.current_stream().cuda_stream
    for i in (1, 6, 7):
        p = f"c{i}_"
        coords, sens, img, y = g[p + "coords"], g[p + "sens"], g[p + "image"], g[p + "y"]
        nx, ny = img.shape
        m, nc = y.shape
        ph0, ph1 = O.build_factors(coords, nx, ny, "single")  # operators.py:72-82
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        t0, t1t, t1c = dev(ph0), dev(ph1.T), dev(np.conj(ph1))
        ts, ti, ty = dev(sens.astype(np.complex64)), dev(img.astype(np.complex64)), \
            dev(y.astype(np.complex64))
        of = torch.empty((m, nc), dtype=torch.complex64, device="cuda")
        oa = torch.empty((nx, ny), dtype=torch.complex64, device="cuda")
        _native.check(lib.csr_nudft_forward_sep(t0.data_ptr(), t1t.data_ptr(), ts.data_ptr(),
                                                ti.data_ptr(), of.data_ptr(), nx, ny, nc, m, st))
        _native.check(lib.csr_nudft_adjoint_sep(t0.data_ptr(), t1c.data_ptr(), ts.data_ptr(),
                                                ty.data_ptr(), oa.data_ptr(), nx, ny, nc, m, st))
        torch.cuda.synchronize()
        assert rel_err(of.cpu().numpy(), g[p + "fwd_double"]) <= 1e-5
        assert rel_err(oa.cpu().numpy(), g[p + "adj_double"]) <= 1e-5
    assert ctypes.sizeof(_native.FactorDesc) > 0
