"""GPU parity of the mixed-order elements (BAR3 quadratic u / linear ebar,
QUAD8 serendipity u / bilinear ebar) against the CPU oracle, through the
C ABI: assembly (CSR structure bit-exact, K and R within the north_star tolerances of
tests/parity.py), defect fields, bitwise run-to-run reproducibility, history, residual norms,
errors, and the paper's 1D bar run with its own discretisation through the GPU Newton loop."""
import numpy as np
import pytest

import oracle
import synth
from paper_2301_06503_b200 import lgdm

from parity import check_records, compare

pytestmark = pytest.mark.gpu

MAT = dict(synth.MATERIAL)


def _mesh(etype, n, distort=0.0, seed=3):
    mesh = synth.mixed_mesh(etype, n, 10.0 * n[0] / 8 if etype == lgdm.QUAD8 else 100.0)
    X = mesh.coords.copy()
    if distort and etype == lgdm.QUAD8:
        h = X[:, 0].max() / n[0]
        corner_ids = np.nonzero(mesh.corner)[0]
        lo, hi = X.min(axis=0), X.max(axis=0)
        inner = np.all((X[corner_ids] > lo + 1e-9) & (X[corner_ids] < hi - 1e-9), axis=1)
        rng = np.random.default_rng(seed)
        X[corner_ids[inner]] += rng.uniform(-1, 1, size=(inner.sum(), 2)) * distort * h
        for c in mesh.conn:
            for k in range(4):
                X[c[4 + k]] = 0.5 * (X[c[k]] + X[c[(k + 1) % 4]])
    return mesh, X


def _gpu(etype, X, conn, dofs, kappa, k0g=None, alg=None, kernel=0, mat_kw=None):
    import torch
    m = lgdm.Mesh(etype, X, conn, lgdm.material(**(mat_kw or MAT)))
    m.set_kernel(kernel)
    m.set_state(dofs, kappa)
    if k0g is not None or alg is not None:
        m.set_defects(k0g, alg)
    out = m.assemble()
    torch.cuda.synchronize()
    got = {q: out[q].torch().cpu().numpy() for q in ("row_ptr", "col_idx", "val", "R")}
    return m, got


CASES = [(lgdm.BAR3, (7,), 0.0), (lgdm.BAR3, (61,), 0.0), (lgdm.QUAD8, (5, 3), 0.0),
         (lgdm.QUAD8, (16, 11), 0.2), (lgdm.QUAD8, (40, 33), 0.1)]


@pytest.mark.parametrize("etype,n,distort", CASES)
@pytest.mark.parametrize("kernel", [0, 1])
def test_mixed_parity(etype, n, distort, kernel):
    mesh, X = _mesh(etype, n, distort)
    dofs, kap = synth.mixed_fields(mesh)
    ref = oracle.mixed_assemble(etype, oracle.material(**MAT), X, mesh.conn, dofs, kap)
    m, got = _gpu(etype, X, mesh.conn, dofs, kap, kernel=kernel)
    assert np.array_equal(m.doff, ref["doff"])
    compare(ref, got, f"mixed {etype} {n}")
    m.close()


@pytest.mark.parametrize("hs,eqv", [(0.0, 0), (30000.0, 1)])
def test_mixed_parity_readings(hs, eqv):
    """reading R2 (h_sigma = 0) and the literal A.3 constants"""
    mesh, X = _mesh(lgdm.QUAD8, (9, 7), 0.15)
    dofs, kap = synth.mixed_fields(mesh)
    kw = dict(MAT, h_sigma=hs, eq_variant=eqv)
    ref = oracle.mixed_assemble(lgdm.QUAD8, oracle.material(**kw), X, mesh.conn, dofs, kap)
    m, got = _gpu(lgdm.QUAD8, X, mesh.conn, dofs, kap, mat_kw=kw)
    compare(ref, got, "readings")
    m.close()


@pytest.mark.parametrize("etype,n", [(lgdm.BAR3, (20,)), (lgdm.QUAD8, (8, 6))])
def test_mixed_parity_defects(etype, n):
    mesh, X = _mesh(etype, n)
    dofs, kap = synth.mixed_fields(mesh)
    ngp = synth.MFAM[etype][3]
    rng = np.random.default_rng(9)
    k0g = MAT["kappa0"] * rng.uniform(0.8, 1.2, size=kap.size)
    alg = rng.uniform(0.9, 0.99, size=kap.size)
    ref = oracle.mixed_assemble(etype, oracle.material(**MAT), X, mesh.conn, dofs, kap,
                                kappa0_gp=k0g, alpha_gp=alg)
    m, got = _gpu(etype, X, mesh.conn, dofs, kap, k0g=k0g, alg=alg)
    compare(ref, got, "defects")
    assert kap.shape[1] == ngp
    m.close()


def test_mixed_bitwise_reproducible():
    mesh, X = _mesh(lgdm.QUAD8, (24, 19), 0.1)
    dofs, kap = synth.mixed_fields(mesh)
    m, a = _gpu(lgdm.QUAD8, X, mesh.conn, dofs, kap)
    import torch
    out = m.assemble()
    torch.cuda.synchronize()
    assert np.array_equal(out["val"].torch().cpu().numpy(), a["val"])
    assert np.array_equal(out["R"].torch().cpu().numpy(), a["R"])
    m.close()


@pytest.mark.parametrize("etype,n", [(lgdm.BAR3, (33,)), (lgdm.QUAD8, (11, 9))])
def test_mixed_history_and_norms(etype, n):
    mesh, X = _mesh(etype, n)
    dofs, kap = synth.mixed_fields(mesh)
    dim = synth.MFAM[etype][0]
    m, got = _gpu(etype, X, mesh.conn, dofs, kap)
    ref = oracle.mixed_assemble(etype, oracle.material(**MAT), X, mesh.conn, dofs, kap)
    kind = oracle.dof_kind(ref["doff"], dim)
    nu, ne = m.residual_norms()
    assert nu == pytest.approx(np.linalg.norm(ref["R"][kind < dim]), rel=1e-10)
    assert ne == pytest.approx(np.linalg.norm(ref["R"][kind == dim]), rel=1e-10)
    m.update_history()
    k_ref = oracle.mixed_update_history(etype, mesh.conn, ref["doff"], dofs, kap)
    # ebar_gp = sum N_a e_a: fused multiply-adds on the GPU, plain products in the oracle
    np.testing.assert_allclose(m.get_kappa().reshape(k_ref.shape), k_ref, rtol=1e-15, atol=0)
    m.close()


def test_mixed_errors():
    mesh, X = _mesh(lgdm.QUAD8, (3, 2))
    bad = mesh.conn.copy()
    bad[0, [1, 4]] = bad[0, [4, 1]]
    with pytest.raises(lgdm.LGDMError) as ei:
        lgdm.Mesh(lgdm.QUAD8, X, bad, lgdm.material(**MAT))
    assert ei.value.status == 1
    inv = mesh.conn.copy()
    inv[0, :4] = inv[0, [1, 0, 3, 2]]                      # clockwise corners
    inv[0, 4:] = inv[0, [4, 7, 6, 5]]
    with pytest.raises(lgdm.LGDMError) as ei:
        lgdm.Mesh(lgdm.QUAD8, X, inv, lgdm.material(**MAT))
    assert ei.value.status == 2
    with pytest.raises(lgdm.LGDMError) as ei:            # slabs need their global dof offset
        lgdm.Mesh(lgdm.QUAD8, X, mesh.conn, lgdm.material(**MAT), global_node_offset=3,
                  n_global_nodes=X.shape[0] + 3)
    assert ei.value.status == 1
    with pytest.raises(lgdm.LGDMError) as ei:            # too few global dofs
        lgdm.Mesh(lgdm.QUAD8, X, mesh.conn, lgdm.material(**MAT), global_dof_offset=0,
                  n_global_dofs=5)
    assert ei.value.status == 1
    dofs, kap = synth.mixed_fields(mesh)
    m, _ = _gpu(lgdm.QUAD8, X, mesh.conn, dofs, kap)
    with pytest.raises(lgdm.LGDMError) as ei:
        m.set_kernel(2)
    assert ei.value.status == 1
    with pytest.raises(lgdm.LGDMError):                   # ebar dof of a corner node
        m.apply_dirichlet([int(m.doff[0]) + 2], [0.0])
    m.close()


def test_bar3_softening_newton_matches_oracle():
    """The paper's 1D bar (Sec. 3.1) with its own discretisation -- quadratic u, linear
    ebar -- and a weaker middle region, displacement-controlled into softening: the GPU
    Newton loop (direct solve) takes the oracle's iteration counts and reaches its reactions and
    history; the reaction peaks then decays and damage localises in the defect."""
    etype, n = lgdm.BAR3, 80
    mesh = synth.mixed_mesh(etype, (n,), 100.0)
    X = mesh.coords
    xc = X[mesh.conn[:, 2], 0]
    L = X[:, 0].max()
    defect = np.abs(xc - L / 2) < 0.05 * L
    k0g = np.repeat(np.where(defect, 0.9, 1.0) * MAT["kappa0"], 3)
    om = oracle.material(**MAT)
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    kind = oracle.dof_kind(doff, 1)
    ids = np.array([doff[0], doff[2 * n]])
    schedule = [(8, 1e-3), (30, 1e-4)]
    nd = int(doff[-1])
    dofs, kh = np.zeros(nd), np.zeros((n, 3))
    its_ref, react_ref = [], []
    for nst, du in schedule:
        inc = np.array([0.0, du])
        for _ in range(nst):
            for it in range(1, 41):
                res = oracle.mixed_assemble(etype, om, X, mesh.conn, dofs, kh, kappa0_gp=k0g)
                delta = oracle.solve(oracle.apply_dirichlet(res, ids, inc if it == 1 else 0 * inc))
                dofs = dofs + delta
                ok, _, _ = oracle.converged_kind(delta, dofs, kind, 1, 1e-6)
                if ok:
                    break
            assert ok
            its_ref.append(it)
            res = oracle.mixed_assemble(etype, om, X, mesh.conn, dofs, kh, kappa0_gp=k0g)
            react_ref.append(oracle.reaction(res, [ids[1]]))
            kh = oracle.mixed_update_history(etype, mesh.conn, doff, dofs, kh)
    m = lgdm.Mesh(etype, X, mesh.conn, lgdm.material(**MAT))
    m.set_state(np.zeros(nd), np.zeros((n, 3)))
    m.set_defects(k0g, None)
    log = []
    for nst, du in schedule:
        log += lgdm.newton(m, ids, [0.0, du], n_steps=nst, tol=1e-6, max_iter=40)
    assert [s["iterations"] for s in log] == its_ref
    r = np.array([s["reaction"] for s in log])
    np.testing.assert_allclose(r, react_ref, rtol=1e-7)
    kap = m.get_kappa().reshape(n, 3)
    np.testing.assert_allclose(kap, kh, rtol=1e-7, atol=1e-14)
    ip = int(r.argmax())
    assert 8 <= ip < len(r) - 5
    assert np.all(np.diff(r[ip:]) < 0)
    kel = kap.max(axis=1)
    assert kel[defect].min() > kel[~defect].max()
    m.close()


def test_mixed_parity_bench_size():
    """the bench.py mixed_order workload (QUAD8 500^2, 250 k elements, 70 M nnz) in full"""
    mesh = synth.mixed_mesh(lgdm.QUAD8, (500, 500), 100.0)
    dofs, kap = synth.mixed_fields(mesh)
    ref = oracle.mixed_assemble(lgdm.QUAD8, oracle.material(**MAT), mesh.coords, mesh.conn,
                                dofs, kap)
    m, got = _gpu(lgdm.QUAD8, mesh.coords, mesh.conn, dofs, kap)
    compare(ref, got, "QUAD8 500^2")
    m.close()


@pytest.mark.parametrize("etype,n,defects", [(lgdm.BAR3, (41,), False), (lgdm.QUAD8, (13, 9), False),
                                             (lgdm.QUAD8, (9, 8), True)])
def test_mixed_update_state(etype, n, defects):
    """state records of Alg. 2 l.8-14 for mixed elements + history commit vs the oracle"""
    mesh, X = _mesh(etype, n, 0.15 if etype == lgdm.QUAD8 else 0.0)
    dofs, kap = synth.mixed_fields(mesh)
    k0g = alg = None
    if defects:
        rng = np.random.default_rng(4)
        k0g = MAT["kappa0"] * rng.uniform(0.8, 1.2, size=kap.size)
        alg = rng.uniform(0.9, 0.99, size=kap.size)
    om = oracle.material(**MAT)
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    sdv_ref, k_ref = oracle.mixed_update_state(etype, om, X, mesh.conn, doff, dofs, kap, k0g, alg)
    m = lgdm.Mesh(etype, X, mesh.conn, lgdm.material(**MAT))
    m.set_state(dofs, kap)
    if defects:
        m.set_defects(k0g, alg)
    out = m.update_state().cpu().numpy()
    assert out.shape == sdv_ref.shape
    check_records(sdv_ref.shape[-1], out, sdv_ref)
    np.testing.assert_allclose(m.get_kappa().reshape(k_ref.shape), k_ref, rtol=1e-15, atol=0)
    m.close()


@pytest.mark.parametrize("etype,n", [(lgdm.BAR3, (9,)), (lgdm.QUAD8, (7, 5)), (lgdm.QUAD8, (40, 31))])
def test_mixed_blocked_order(etype, n):
    """the paper's [u; ebar] order of a mixed system: bit-identical values"""
    import torch
    mesh, X = _mesh(etype, n, 0.1 if etype == lgdm.QUAD8 else 0.0)
    dofs, kap = synth.mixed_fields(mesh)
    m, got = _gpu(etype, X, mesh.conn, dofs, kap)
    b = m.get_blocked()
    torch.cuda.synchronize()
    gb = {q: b[q].torch().cpu().numpy() for q in ("row_ptr", "col_idx", "val", "R")}
    dim = synth.MFAM[etype][0]
    p = oracle.mixed_blocked_perm(m.doff, dim)
    ref = oracle.blocked_from_perm(dict(got, col_idx=got["col_idx"].astype(np.int32)), p)
    for q in ("row_ptr", "col_idx", "val", "R"):
        assert np.array_equal(gb[q], ref[q]), q
    m.close()


def test_quad8_strip_newton_matches_oracle():
    """2D with the paper's own discretisation (serendipity u, bilinear ebar): a plane
    strain strip pulled at x = L with a weaker column of elements, three displacement steps
    into damage; the GPU Newton loop (direct solve) matches the oracle's iteration counts,
    reactions and committed history."""
    etype, n = lgdm.QUAD8, (8, 3)
    mesh = synth.mixed_mesh(etype, n, 8.0)
    X = mesh.coords
    ne = mesh.conn.shape[0]
    ex = X[mesh.conn[:, :4], 0].mean(axis=1)
    k0g = np.repeat(np.where(np.abs(ex - 4.0) < 0.6, 0.9, 1.0) * MAT["kappa0"], 9)
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    kind = oracle.dof_kind(doff, 2)
    left = np.nonzero(X[:, 0] == X[:, 0].min())[0]
    right = np.nonzero(X[:, 0] == X[:, 0].max())[0]
    ids = np.concatenate([doff[left], doff[left] + 1, doff[right]])
    inc = np.concatenate([np.zeros(2 * left.size), np.full(right.size, 1.0)])
    om = oracle.material(**MAT)
    nd = int(doff[-1])
    schedule = [(2, 3e-4), (3, 1e-4)]
    dofs, kh = np.zeros(nd), np.zeros((ne, 9))
    its_ref, react_ref = [], []
    for nst, du in schedule:
        for _ in range(nst):
            for it in range(1, 41):
                res = oracle.mixed_assemble(etype, om, X, mesh.conn, dofs, kh, kappa0_gp=k0g)
                delta = oracle.solve(oracle.apply_dirichlet(res, ids, inc * du if it == 1 else 0 * inc))
                dofs = dofs + delta
                ok, _, _ = oracle.converged_kind(delta, dofs, kind, 2, 1e-6)
                if ok:
                    break
            assert ok
            its_ref.append(it)
            res = oracle.mixed_assemble(etype, om, X, mesh.conn, dofs, kh, kappa0_gp=k0g)
            react_ref.append(oracle.reaction(res, doff[right]))
            kh = oracle.mixed_update_history(etype, mesh.conn, doff, dofs, kh)
    assert kh.max() > MAT["kappa0"]                       # the run reaches damage
    m = lgdm.Mesh(etype, X, mesh.conn, lgdm.material(**MAT))
    m.set_state(np.zeros(nd), np.zeros((ne, 9)))
    m.set_defects(k0g, None)
    log = []
    for nst, du in schedule:
        log += lgdm.newton(m, ids, inc * du, n_steps=nst, tol=1e-6, max_iter=40)
    assert [s["iterations"] for s in log] == its_ref
    np.testing.assert_allclose([s["reaction"] for s in log], react_ref, rtol=1e-7)
    np.testing.assert_allclose(m.get_kappa().reshape(kh.shape), kh, rtol=1e-7, atol=1e-14)
    m.close()


@pytest.mark.parametrize("etype,n,P", [(lgdm.QUAD8, (12, 9), 3), (lgdm.BAR3, (30,), 2)])
def test_mixed_slabs_stitch_bitwise(etype, n, P):
    """slab rows (ghost elements recomputed, global dof columns) equal the whole mesh's rows
    bitwise (SURVEY 8e for the mixed-order elements)"""
    from paper_2301_06503_b200 import slabs as sl
    mesh = synth.mixed_mesh(etype, n, 10.0)
    doff = oracle.mixed_dofs(etype, mesh.coords.shape[0], mesh.conn)
    dofs, kap = synth.mixed_fields(mesh)
    mw, whole = _gpu(etype, mesh.coords, mesh.conn, dofs, kap)
    rp = whole["row_ptr"]
    covered = 0
    import torch
    for p in range(P):
        S = sl.mixed_slab(etype, n, p, P)
        (nb, ne_), (eb, ee), (ob, oe) = S.node_range, S.elem_range, S.owned_local
        assert S.global_dof_offset == doff[nb] and S.n_global_dofs == doff[-1]
        conn = mesh.conn[eb:ee] - nb
        assert conn.min() >= 0 and conn.max() < ne_ - nb
        m = lgdm.Mesh(etype, mesh.coords[nb:ne_], conn, lgdm.material(**MAT),
                      global_node_offset=int(nb), n_global_nodes=mesh.coords.shape[0],
                      owned=(int(ob), int(oe)), global_dof_offset=S.global_dof_offset,
                      n_global_dofs=S.n_global_dofs)
        m.set_state(dofs[doff[nb]:doff[ne_]], kap[eb:ee])
        out = m.assemble()
        torch.cuda.synchronize()
        r0, r1 = int(doff[nb + ob]), int(doff[nb + oe])
        assert out["first_row"] == r0 and out["n_cols"] == doff[-1] and out["n_rows"] == r1 - r0
        grp = out["row_ptr"].torch().cpu().numpy()
        assert np.array_equal(grp, rp[r0:r1 + 1] - rp[r0])
        assert np.array_equal(out["col_idx"].torch().cpu().numpy(), whole["col_idx"][rp[r0]:rp[r1]])
        assert np.array_equal(out["val"].torch().cpu().numpy(), whole["val"][rp[r0]:rp[r1]])
        assert np.array_equal(out["R"].torch().cpu().numpy(), whole["R"][r0:r1])
        covered += r1 - r0
        m.close()
    assert covered == doff[-1]
    mw.close()


def test_sen2d_newton_physics():
    """The paper's 2D side-edge-notch setting (SPEC default geometry: 100 mm plate,
    50 mm mid-height edge slit) with its QUAD8 discretisation through the GPU Newton loop
    (reading R2): damage starts next to the notch tip, the most damaged elements lie along the
    ligament (y = 50 mm, x > 50 mm), and the load-displacement curve has a single peak followed
    by softening."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "sen2d", os.path.join(os.path.dirname(__file__), "..", "tools", "sen2d.py"))
    sen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sen)
    mesh, log, r, kap = sen.run(n=16, steps=70, du=2e-4, tol=1e-5, verbose=False)
    X = mesh.coords
    c = X[mesh.conn[:, :4]].mean(axis=1)
    k = kap.max(axis=1)
    h = 100.0 / 16
    worst = c[np.argsort(k)[-4:]]
    assert np.all(np.abs(worst[:, 1] - 50.0) < h)            # on the ligament row
    assert np.all(worst[:, 0] > 50.0 - 1e-9)                  # ahead of the notch tip
    tip = c[int(k.argmax())]
    assert abs(tip[0] - 50.0) < 2 * h                         # the tip element is the worst
    ip = int(r.argmax())
    assert 5 < ip < len(r) - 5
    assert r[-1] < 0.8 * r.max()
    assert np.all(np.diff(r[:ip]) > 0)
