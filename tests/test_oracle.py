"""The CPU oracle (oracle/spk_oracle.c) pinned against vectors produced by the reference
itself (tests/golden/make_golden.py).  Bitwise wherever the reference is deterministic
numba code; tolerance only against the reference's FFT (precompute_field)."""

import numpy as np
import pytest

from oracle import oracle as orc
from spk_golden import golden


@pytest.fixture(scope="module")
def rep():
    return golden("repulsion")


@pytest.fixture(scope="module")
def proj():
    return golden("projection")


@pytest.fixture(scope="module")
def att():
    return golden("attraction")


def test_direct_sums_bitwise(rep):
    # _treecode.direct_sums (_treecode.py:506-534)
    for name in rep["names"]:
        val, grad = orc.direct_sums(rep[f"{name}_pos"], float(rep[f"{name}_eps2"]))
        assert np.array_equal(val, rep[f"{name}_val"]), name
        assert np.array_equal(grad, rep[f"{name}_grad"]), name


def test_normalised_repulsion_bitwise(rep):
    # eval_repulsion_direct normalisation (repulsion.py:72-87)
    for name in rep["names"]:
        eps = float(np.sqrt(rep[f"{name}_eps2"]))
        cost, grad = orc.repulsion(rep[f"{name}_pos"], eps)
        assert cost == float(rep[f"{name}_cost"]), name
        assert np.array_equal(grad, rep[f"{name}_gnorm"]), name


def test_direct_sums_subset_bitwise(rep):
    val, grad = orc.direct_sums_subset(rep["spokes3d_pos"], rep["subset_targets"], 1e-6)
    assert np.array_equal(val, rep["subset_val"])
    assert np.array_equal(grad, rep["subset_grad"])


def test_two_particle_hand_values():
    # tests/test_repulsion.py:23-29 in the reference
    cost, grad = orc.repulsion(np.array([[0.0, 0, 0], [1.0, 0, 0]]), 0.0)
    assert abs(cost - 0.25) < 1e-12
    assert np.abs(grad - np.array([[-0.25, 0, 0], [0.25, 0, 0]])).max() < 1e-12


def test_grid_sums_equal_precompute_field_at_nodes(att):
    # The exact weighted sum at the nodes is precompute_field's linear convolution
    # (attraction.py:62-113); FFT rounding only.
    for name in att["names"]:
        rho = att[f"{name}_rho"]
        n = int(att[f"{name}_n"])
        d = rho.ndim
        axis = np.arange(-n, n + 1, dtype=np.float64) / n
        nodes = np.stack(np.meshgrid(*([axis] * d), indexing="ij"), -1).reshape(-1, d)
        eps = float(att[f"{name}_eps"])
        val, grad = orc.grid_sums(nodes, rho, eps * eps)
        pot = att[f"{name}_potential"].reshape(-1)
        force = att[f"{name}_force"].reshape(d, -1).T
        assert np.abs(val - pot).max() <= 1e-12 * np.abs(pot).max(), name
        assert np.abs(grad - force).max() <= 1e-11 * max(np.abs(force).max(), 1e-300), name


def _case(proj, name):
    return dict(a=float(proj[f"{name}_a"]), b=float(proj[f"{name}_b"]),
                pin=int(proj[f"{name}_pin"]), pv=proj[f"{name}_pinval"],
                npit=int(proj[f"{name}_npit"]), tau=1.0 / float(proj[f"{name}_lam"]),
                mono=bool(proj[f"{name}_mono"]), tol=float(proj[f"{name}_tol"]))


def test_fista_bitwise(proj):
    # _project_shot (projection.py:169-284), no polish
    for name in proj["names"]:
        c = _case(proj, name)
        shots = proj[f"{name}_in"]
        for s in range(shots.shape[0]):
            out, _ = orc.project_shot(shots[s], c["a"], c["b"], c["pin"], c["pv"], c["npit"],
                                      c["tau"], c["mono"])
            assert np.array_equal(out, proj[f"{name}_fista"][s]), (name, s)


def test_project_all_bitwise(proj):
    # _project_all (projection.py:376-382): FISTA + polish
    for name in proj["names"]:
        c = _case(proj, name)
        out, _ = orc.project_all(proj[f"{name}_in"], c["a"], c["b"], c["pin"], c["pv"],
                                 c["npit"], c["tau"], c["tol"], monotone=c["mono"])
        assert np.array_equal(out, proj[f"{name}_out"]), name


def test_project_all_nonfinite_bitwise():
    # NaN / +-inf samples through _project_all (numba kernel fixture): NaN spreads and
    # the polish's comparisons treat it as satisfied, exactly as in the reference
    nf = golden("projection_nonfinite")
    for name in nf["names"]:
        out, _ = orc.project_all(nf[f"{name}_in"], float(nf[f"{name}_a"]),
                                 float(nf[f"{name}_b"]), int(nf[f"{name}_pin"]),
                                 nf[f"{name}_pinval"], 50, 1.0 / float(nf[f"{name}_lam"]), 1e-7)
        assert np.isnan(out).any(), name
        assert np.array_equal(out, nf[f"{name}_out"], equal_nan=True), name


def test_trace_bitwise(proj):
    for name in ("mono2d", "trace3d"):
        c = _case(proj, name)
        _, trace, _ = orc.project_shot(proj[f"{name}_in"][0], c["a"], c["b"], c["pin"],
                                       c["pv"], c["npit"], c["tau"], c["mono"],
                                       return_trace=True)
        assert np.array_equal(trace, proj[f"{name}_trace"]), name


def test_polish_bitwise_and_capped(proj):
    a, b, pin = float(proj["polish_a"]), float(proj["polish_b"]), int(proj["polish_pin"])
    for s in range(proj["polish_in"].shape[0]):
        out, sweeps = orc.polish(proj["polish_in"][s], a, b, pin, np.zeros(3), 1e-7)
        assert np.array_equal(out, proj["polish_out"][s])
        assert sweeps > 32  # exercises many wavefront batches on the GPU side
        capped, n = orc.polish(proj["polish_in"][s], a, b, pin, np.zeros(3), 1e-7, 37)
        assert n == 37
        assert np.array_equal(capped, proj["polish_capped37"][s])


def test_anisotropic_grid_sums_match_cubic_when_isotropic():
    # The anisotropic oracle path reduces to the cubic one when all N_a agree.
    rng = np.random.default_rng(3)
    rho = rng.uniform(0, 1, (9, 9, 9))
    rho /= rho.sum()
    pts = rng.uniform(-1, 1, (20, 3))
    v1, g1 = orc.grid_sums(pts, rho, 1e-3)
    # an explicit O(G) restatement with node coordinates (i - N)/N
    ax = (np.arange(9) - 4) / 4.0
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    for t in range(3):
        d = pts[t][:, None, None, None] - np.stack([X, Y, Z])
        h = np.sqrt(1e-3 + (d * d).sum(0))
        assert abs(v1[t] - (rho * h).sum()) <= 1e-12 * v1[t]
        assert np.abs(g1[t] - (rho * d / h).reshape(3, -1).sum(1)).max() <= 1e-12


def test_projection_oracle_solves_the_qp():
    """The oracle's FISTA + polish at n_pit=1000 vs an independent QP solve (SLSQP) of the
    reference's acceptance-test problem (test_acceptance.py:153-173): <= 1e-4 there,
    measured ~2e-7."""
    from paper_2108_02991_b200.projection import stacked_operator_norm
    from qp_ref import qp_reference

    rng = np.random.default_rng(7)
    a, b = 0.3, 0.15
    tau = 1.0 / stacked_operator_norm(8, -1)
    for _ in range(20):
        shot = rng.uniform(-1.5, 1.5, (8, 2))
        out, _ = orc.project_all(shot[None], a, b, -1, np.zeros(2), 1000, tau, 1e-7)
        assert np.abs(out[0] - qp_reference(shot, a, b)).max() <= 1e-5
