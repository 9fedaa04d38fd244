"""The reference's solver-level known-answer tests on the device kernels (GPU box).

kd_padmm_solve_batched (build_backend + padmm_solve) and kd_cr_solve_batched
(bake_jacobian + cr_solve) run the same dense / CR kernels as a batch step on
pre-assembled systems, so the reference's unit tests of those functions can
run against the device:

* test_padmm.cpp:201-293 — zero v_f converges in one iteration; a
  bilateral-only system solves D lambda = -v_f; the solution is invariant in
  eta and rho; without acceleration the combined residual is non-increasing;
  fixed-iteration mode runs exactly max_iters (also on a zero problem);
* test_delassus.cpp:192-245, 305-320 — cr_solve returns an exact warm start
  unchanged (breakdown, 0 iterations); one iteration on a uniform diagonal;
  at most n_distinct iterations on a diagonal; monotone residual history;
  dense and matrix-free agree with a generous budget.

The chain problem (test_padmm.cpp:35-54) is serial_chain_10 at its initial
pose, assembled by the oracle (its rows equal the device's to 1e-12, see
test_parity_gpu.py); the system matrices for the direct-solve checks are built
here in numpy.
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(4242)


def _quat_R(q):
    w, x, y, z = np.asarray(q, float) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _inertias(sc):
    """world_inertias (delassus.cpp:21-34) at the scene's initial poses."""
    im, iw = [], []
    for b in sc.bodies:
        R = _quat_R(b.orientation)
        I = R @ np.asarray(b.inertia, float) @ R.T
        I = 0.5 * (I + I.T)
        inv = np.linalg.inv(I)
        im.append(1.0 / b.mass)
        iw.append(0.5 * (inv + inv.T))
    return np.array(im), np.array(iw)


def _rows(sc):
    """The ConstraintSet at the initial pose and v_f = J u_free - v* (the
    oracle's first-step rows; StepConfig defaults, so AssembleConfig{})."""
    ob = oracle_lib.OracleBatch([oracle_lib.OracleModel(sc)], [0], n_threads=1)
    ob.set_trace(True)
    ob.step(K.StepConfig())
    r = ob.dump_rows(0)
    return r, r["vf"] / r["scale"]


def chain_problem():
    sc = oracle_lib.bundled_scene("serial_chain_10")
    r, vf = _rows(sc)
    im, iw = _inertias(sc)
    return sc, r, vf, im, iw


def _problem(r, im, iw, scale, rhs, reg=None, **kw):
    return K.SolveProblem(body=r["body"], jacobian=r["J"], reg=r["reg"] if reg is None else reg, scale=scale,
                          inv_mass=im, inv_inertia=iw, rhs=rhs, **kw)


def _dense_D(r, im, iw, scale, eta_rho):
    """P (J M^-1 J^T + R) P + eta_rho I from full matrices (the naive oracle of
    test_delassus.cpp:26-40)."""
    n, nb = len(r["reg"]), len(im)
    J = np.zeros((n, 6 * nb))
    for i in range(n):
        for side in range(2):
            b = r["body"][i, side]
            if b >= 0:
                J[i, 6 * b:6 * b + 6] += r["J"][i, 6 * side:6 * side + 6]
    Minv = np.zeros((6 * nb, 6 * nb))
    for b in range(nb):
        Minv[6 * b:6 * b + 3, 6 * b:6 * b + 3] = im[b] * np.eye(3)
        Minv[6 * b + 3:6 * b + 6, 6 * b + 3:6 * b + 6] = iw[b]
    D = J @ Minv @ J.T + np.diag(r["reg"])
    return np.diag(scale) @ D @ np.diag(scale) + eta_rho * np.eye(n)


@pytest.mark.parametrize("backend", ["dense", "sparse"])
def test_zero_free_velocity_converges_in_one_iteration(backend):
    _, r, vf, im, iw = chain_problem()
    n = len(vf)
    cfg = K.StepConfig()
    out = K.padmm_solve([_problem(r, im, iw, np.ones(n), np.zeros(n))], cfg.eta + cfg.rho, cfg, backend=backend)[0]
    assert np.linalg.norm(out["lambda"]) == 0.0
    assert out["diag"].iterations == 1 and out["diag"].converged


@pytest.mark.parametrize("backend,budget", [("dense", 9), ("sparse", 60)])
def test_bilateral_system_solves_D_lambda_eq_minus_vf(backend, budget):
    _, r, vf, im, iw = chain_problem()
    cfg = K.StepConfig(eps=1e-10, max_iters=2000)
    P = r["scale"]
    out = K.padmm_solve([_problem(r, im, iw, P, P * vf)], cfg.eta + cfg.rho, cfg, backend=backend,
                        cr_budget=budget)[0]
    assert out["diag"].converged
    lam = P * out["lambda"]
    expected = np.linalg.solve(_dense_D(r, im, iw, np.ones(len(P)), 0.0), -vf)
    assert np.abs(lam - expected).max() / max(1.0, np.abs(expected).max()) < 1e-6


def test_solution_invariant_in_eta_and_rho_batched():
    """The three (eta, rho) pairs of test_padmm.cpp:235-258, one device call each
    (eta_rho is per call), each call a batch of the same problem twice."""
    _, r, vf, im, iw = chain_problem()
    P = r["scale"]
    sols = []
    for eta, rho in ((1e-5, 0.1), (1e-5, 1.0), (1e-3, 1.0)):
        cfg = K.StepConfig(eta=eta, rho=rho, eps=1e-9, max_iters=5000)
        outs = K.padmm_solve([_problem(r, im, iw, P, P * vf)] * 2, eta + rho, cfg, backend="dense")
        for o in outs:
            assert o["diag"].converged
        assert np.array_equal(outs[0]["lambda"], outs[1]["lambda"])  # worlds are independent
        sols.append(P * outs[0]["lambda"])
    scale = max(1.0, np.abs(sols[0]).max())
    assert np.abs(sols[0] - sols[1]).max() / scale < 1e-5
    assert np.abs(sols[0] - sols[2]).max() / scale < 1e-5


def test_without_acceleration_the_residual_is_non_increasing():
    _, r, vf, im, iw = chain_problem()
    cfg = K.StepConfig(acceleration=False, restart=False, eps=1e-12, max_iters=400)
    P = r["scale"]
    h = K.padmm_solve([_problem(r, im, iw, P, P * vf)], cfg.eta + cfg.rho, cfg, backend="dense",
                      history_capacity=400)[0]["history"]
    assert len(h) > 2
    assert np.all(h[1:] <= h[:-1] + 1e-12)


def test_fixed_iteration_mode_runs_exactly_max_iters():
    _, r, vf, im, iw = chain_problem()
    cfg = K.StepConfig(fixed_iteration_mode=True, max_iters=17)
    P = r["scale"]
    n = len(P)
    outs = K.padmm_solve([_problem(r, im, iw, P, P * vf), _problem(r, im, iw, P, np.zeros(n))], cfg.eta + cfg.rho,
                         cfg, backend="dense", history_capacity=32)
    assert outs[0]["diag"].iterations == 17 and len(outs[0]["history"]) == 17
    assert outs[1]["diag"].iterations == 17 and outs[1]["diag"].converged


def test_padmm_matches_oracle_history_on_contacts():
    """A contact system (sphere on the plane, one SOC triple): the device's
    residual history equals the oracle step's (fixed mode, 12 iterations)."""
    sc = oracle_lib.bundled_scene("sphere_on_plane")
    cfg = K.StepConfig(fixed_iteration_mode=True, max_iters=12)
    ob = oracle_lib.OracleBatch([oracle_lib.OracleModel(sc)], [0], n_threads=1)
    ob.set_trace(True)
    ob.step(cfg)
    r = ob.dump_rows(0)
    d = ob.diagnostics()[0]
    im, iw = _inertias(sc)
    _, cd = ob.dump_contacts(0)
    mu = cd[:, 7]
    prob = _problem(r, im, iw, r["scale"], r["vf"], n_bilateral=d.first_contact_row - d.n_limits,
                    n_limits=d.n_limits, n_contacts=d.contact_count, mu=mu)
    out = K.padmm_solve([prob], cfg.eta + cfg.rho, cfg, backend="dense", history_capacity=16)[0]
    ho = ob.history(16)[0][:12]
    assert np.all(np.abs(out["history"] - ho) <= 1e-9 * np.maximum(1e-3, np.abs(ho)) + 1e-13)
    assert np.abs(out["lambda"] - r["lambda"]).max() / max(1.0, np.abs(r["lambda"]).max()) < 1e-9


def _diag_problem(diag, rhs, x0=None):
    n = len(diag)
    return K.SolveProblem(body=-np.ones((n, 2), np.int32), jacobian=np.zeros((n, 12)), reg=np.asarray(diag, float),
                          scale=np.ones(n), inv_mass=np.ones(1), inv_inertia=np.eye(3)[None], rhs=rhs, x0=x0)


def test_cr_returns_an_exact_warm_start_unchanged():
    rhs = RNG.uniform(-1, 1, 4)
    out = K.cr_solve([_diag_problem([2.0] * 4, rhs, x0=rhs / 2.0)], 0.0, 10)[0]
    assert np.abs(out["x"] - rhs / 2.0).max() == 0.0
    assert out["breakdown"] and out["iterations"] == 0


def test_cr_one_iteration_on_a_uniform_diagonal():
    rhs = RNG.uniform(-1, 1, 6)
    out = K.cr_solve([_diag_problem([3.0] * 6, rhs)], 0.0, 1, history_capacity=4)[0]
    assert np.abs(out["x"] - rhs / 3.0).max() < 1e-14
    assert len(out["history"]) == 2


def test_cr_at_most_n_distinct_iterations_on_a_diagonal():
    d = np.array([1, 1, 2, 2, 2, 5, 5, 1], float)
    rhs = RNG.uniform(-1, 1, 8)
    out = K.cr_solve([_diag_problem(d, rhs)], 0.0, 3)[0]
    assert np.abs(d * out["x"] - rhs).max() < 1e-10


def test_cr_residual_norm_is_monotone():
    _, r, _, im, iw = chain_problem()
    rhs = RNG.uniform(-1, 1, len(r["reg"]))
    out = K.cr_solve([_problem(r, im, iw, r["scale"], rhs)], 1.0, 40, history_capacity=64)[0]
    h = out["history"]
    assert len(h) >= 2 and np.all(h[1:] <= h[:-1] + 1e-12)


def test_dense_and_matrix_free_backends_agree():
    sc = oracle_lib.bundled_scene("fourbar")
    r, _ = _rows(sc)
    im, iw = _inertias(sc)
    n = len(r["reg"])
    D = _dense_D(r, im, iw, np.ones(n), 1.0)
    rhss = [RNG.uniform(-1, 1, n) for _ in range(5)]
    outs = K.cr_solve([_problem(r, im, iw, np.ones(n), b) for b in rhss], 1.0, 200)
    for b, o in zip(rhss, outs):
        xd = np.linalg.solve(D, b)
        assert np.abs(xd - o["x"]).max() < 1e-6 * max(1.0, np.abs(xd).max())


def test_batch_assemble_equals_oracle_rows_and_leaves_state():
    """kd_batch_assemble = assemble_constraints on the device: the rows of the
    current state (oracle's first-step rows) and no change to the state."""
    from paper_2603_16536_b200.scenes import dr_legs
    sc = dr_legs()
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    gb = K.WorldBatch()
    gb.add_world(m)
    p0, t0, _ = gb.get_state()
    gb.assemble(cfg)
    p1, t1, _ = gb.get_state()
    assert np.array_equal(p0, p1) and np.array_equal(t0, t1)
    ob = oracle_lib.OracleBatch([oracle_lib.OracleModel(sc)], [0], n_threads=1)
    ob.set_trace(True)
    ob.step(cfg)
    rg, ro = gb.dump_rows(0), ob.dump_rows(0)
    assert (rg["body"] == ro["body"]).all() and (rg["kind"] == ro["kind"]).all()
    for key in ("J", "bias", "reg", "scale", "vf"):
        assert np.abs(rg[key] - ro[key]).max() / max(1.0, np.abs(ro[key]).max()) < 1e-12, key
    cg, _ = gb.dump_contacts(0)
    co, _ = ob.dump_contacts(0)
    assert (cg == co).all()
