"""Pins of the oracle's Newton pieces (SPEC.md solver module) -- CPU.

Pinned against: SPEC's elimination examples (no constraints -> unchanged; a constrained dof
solves to its increment exactly, 0 on subsequent iterations), the exact linear solution of an
elastic 1D bar under an end displacement (u = d x / L after one iteration), the dense solve,
and the convergence-check examples.
"""
import numpy as np
import pytest

import oracle
import synth


def _bar(n, kappa0=1.0):
    cfg = synth.small_config(oracle.BAR2, (n,))
    mesh = synth.structured_mesh(cfg)
    mat = dict(synth.MATERIAL)
    mat["kappa0"] = kappa0          # damage never triggers (elastic limit, SPEC example)
    return cfg, mesh, oracle.material(**mat)


def test_no_constraints_unchanged():
    cfg, mesh, m = _bar(4)
    d, k = synth.fields(cfg, mesh)
    res = oracle.assemble(oracle.BAR2, m, mesh.coords, mesh.conn, d, k)
    out = oracle.apply_dirichlet(res, [], [])
    assert np.array_equal(out["val"], res["val"]) and np.array_equal(out["R"], res["R"])


@pytest.mark.parametrize("first", [True, False])
def test_constrained_dof_solves_to_increment(first):
    cfg, mesh, m = _bar(6)
    d, k = synth.fields(cfg, mesh)
    d = d * 0.1
    fixed = [0, 2 * 6]                      # u of the two end nodes
    incr = [0.0, 0.25e-3 if first else 0.0]
    res = oracle.assemble(oracle.BAR2, m, mesh.coords, mesh.conn, d, k)
    delta = oracle.solve(oracle.apply_dirichlet(res, fixed, incr))
    assert delta[fixed[0]] == 0.0 and delta[fixed[1]] == incr[1]


def test_elastic_bar_one_iteration_is_exact():
    """virgin bar, u(0) = 0, u(L) = d: one Newton iteration gives u = d x / L (linear FE
    reproduce it exactly) and ebar solves the Helmholtz-type equation with eeq = d / L"""
    n = 8
    cfg, mesh, m = _bar(n)
    L = mesh.coords[-1, 0] - mesh.coords[0, 0]
    dofs = np.zeros(2 * (n + 1))
    kap = np.full(n * 2, 0.0)
    dd = 1e-3
    delta, new = oracle.newton_iteration(oracle.BAR2, m, mesh.coords, mesh.conn, dofs, kap,
                                         [0, 2 * n], [0.0, dd])
    u = new.reshape(-1, 2)[:, 0]
    np.testing.assert_allclose(u, dd * (mesh.coords[:, 0] - mesh.coords[0, 0]) / L, rtol=1e-12,
                               atol=1e-18)
    # second iteration: the residual of the linear problem is zero -> delta = 0 (SPEC: "second
    # confirms")
    delta2, _ = oracle.newton_iteration(oracle.BAR2, m, mesh.coords, mesh.conn, new, kap,
                                        [0, 2 * n], [0.0, 0.0])
    assert np.abs(delta2).max() <= 1e-12 * np.abs(new).max()


def test_solve_matches_dense():
    cfg = synth.small_config(oracle.QUAD4, (3, 3))
    mesh = synth.structured_mesh(cfg)
    d, k = synth.fields(cfg, mesh)
    m = oracle.material(**synth.MATERIAL)
    res = oracle.assemble(oracle.QUAD4, m, mesh.coords, mesh.conn, d, k)
    fixed = [0, 1, 3 * 3, 3 * 3 + 1]
    sys_ = oracle.apply_dirichlet(res, fixed, [0.0] * 4)
    n = sys_["R"].size
    K = np.zeros((n, n))
    for i in range(n):
        for q in range(sys_["row_ptr"][i], sys_["row_ptr"][i + 1]):
            K[i, sys_["col_idx"][q]] = sys_["val"][q]
    np.testing.assert_allclose(oracle.solve(sys_), np.linalg.solve(K, sys_["R"]), rtol=1e-9,
                               atol=1e-14 * np.abs(sys_["R"]).max())


def test_convergence_check_examples():
    et = oracle.QUAD4
    u = np.ones(12)
    assert oracle.converged(et, np.zeros(12), u, 1e-4)[0]
    d = np.zeros(12)
    d[0] = 2e-4 * np.linalg.norm(u.reshape(-1, 3)[:, :2])
    assert not oracle.converged(et, d, u, 1e-4)[0]
    assert oracle.converged(et, np.zeros(12), np.zeros(12), 1e-4)[0]     # floor guard


def test_reaction_elastic_bar():
    """SPEC reaction_force example: elastic 1D bar, applied end displacement u -> E A u / L"""
    n = 10
    cfg, mesh, m = _bar(n)
    L = mesh.coords[-1, 0] - mesh.coords[0, 0]
    dofs = np.zeros(2 * (n + 1))
    kap = np.zeros(2 * n)
    d = 2e-4
    _, new = oracle.newton_iteration(oracle.BAR2, m, mesh.coords, mesh.conn, dofs, kap, [0, 2 * n],
                                     [0.0, d])
    res = oracle.assemble(oracle.BAR2, m, mesh.coords, mesh.conn, new, kap)
    E, A = synth.MATERIAL["E"], synth.MATERIAL["t"]
    assert oracle.reaction(res, [2 * n]) == pytest.approx(E * A * d / L, rel=1e-10)
    assert oracle.reaction(res, [0]) == pytest.approx(-E * A * d / L, rel=1e-10)
    assert oracle.reaction(oracle.assemble(oracle.BAR2, m, mesh.coords, mesh.conn, dofs, kap),
                           [2 * n]) == 0.0
