"""Pins of the mixed-order oracle (quadratic u with linear ebar, the paper's
own discretisation) -- CPU only.

Pins: shape functions by their interpolation properties (Kronecker delta at the nodes,
partition of unity, reproduction of complete quadratics / linears, derivatives by central
differences) -- which determine them uniquely; the 3-point Gauss rule on monomials; whole
element blocks and residuals in undamaged states against exact symbolic integration (sympy,
shape functions rebuilt from a Vandermonde solve, not retyped); the damaged constant state
of the bar in closed form; QUAD8 ebar blocks equal to the (separately pinned) Q4 oracle's
where both quadratures are exact; the patch test on distorted QUAD8 patches; rigid-body
null space, symmetry and exact nullity; central finite differences of R against K in
damaged states; the pattern and the assembly against brute force; the history update.
"""
import numpy as np
import pytest
import sympy as sp

import oracle
import synth

MAT = dict(synth.MATERIAL)
BAR3, QUAD8 = 4, 5


def mat(**kw):
    d = dict(MAT)
    d.update(kw)
    return oracle.material(**d)


def ref_nodes(etype):
    if etype == BAR3:
        return np.array([[-1.0], [1.0], [0.0]])
    return np.array([[-1, -1], [1, -1], [1, 1], [-1, 1], [0, -1], [1, 0], [0, 1], [-1, 0]],
                    dtype=np.float64)


def ldof(etype, a):
    dim, nenu, nene = oracle.mixed_family(etype)[:3]
    return a * (dim + 1) if a < nene else nene * (dim + 1) + (a - nene) * dim


def dense(res, n):
    K = np.zeros((n, n))
    rp, ci, v = res["row_ptr"], res["col_idx"], res["val"]
    for r in range(n):
        K[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    return K


# ---------------- shape functions and Gauss rule ----------------

@pytest.mark.parametrize("etype", [BAR3, QUAD8])
def test_shape_interpolation(etype):
    dim, nenu, nene = oracle.mixed_family(etype)[:3]
    XR = ref_nodes(etype)
    for b in range(nenu):                                  # Kronecker delta at the u nodes
        N, _ = oracle.mixed_shape(etype, XR[b], "u")
        np.testing.assert_allclose(N, np.eye(nenu)[b], atol=1e-15)
    for b in range(nene):                                  # ... and at the corners for ebar
        N, _ = oracle.mixed_shape(etype, XR[b], "e")
        np.testing.assert_allclose(N, np.eye(nene)[b], atol=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(10):
        p = rng.uniform(-1, 1, size=dim)
        for field, nen in (("u", nenu), ("e", nene)):
            N, dN = oracle.mixed_shape(etype, p, field)
            X = XR[:nen]
            assert N.sum() == pytest.approx(1.0, rel=1e-15)
            np.testing.assert_allclose(N @ X, p, atol=1e-15)          # linear completeness
            np.testing.assert_allclose(dN.T @ X, np.eye(dim), atol=1e-14)
            if field == "u":                                          # quadratic completeness
                assert N @ X[:, 0] ** 2 == pytest.approx(p[0] ** 2, abs=1e-15)
                if dim == 2:
                    assert N @ (X[:, 0] * X[:, 1]) == pytest.approx(p[0] * p[1], abs=1e-15)
                    assert N @ X[:, 1] ** 2 == pytest.approx(p[1] ** 2, abs=1e-15)
            for k in range(dim):                                      # central differences
                e = np.zeros(dim)
                e[k] = 1e-6
                fd = (oracle.mixed_shape(etype, p + e, field)[0] -
                      oracle.mixed_shape(etype, p - e, field)[0]) / 2e-6
                np.testing.assert_allclose(dN[:, k], fd, atol=1e-9)


@pytest.mark.parametrize("etype", [BAR3, QUAD8])
def test_gauss3(etype):
    dim = oracle.mixed_family(etype)[0]
    xi, w = oracle.mixed_gauss(etype)
    exact = {0: 2.0, 1: 0.0, 2: 2.0 / 3.0, 3: 0.0, 4: 2.0 / 5.0, 5: 0.0}
    for p in range(6):                                   # 3 points: exact to degree 5 per axis
        for q in (range(6) if dim == 2 else [0]):
            v = (w * xi[:, 0] ** p * (xi[:, 1] ** q if dim == 2 else 1.0)).sum()
            assert v == pytest.approx(exact[p] * (exact[q] if dim == 2 else 1.0), abs=1e-15)


# ---------------- exact symbolic element (undamaged states) ----------------

def _sym_shapes(etype, a_len, b_len):
    """u and ebar shape functions on the physical element [0,a] (x [0,b]) by Vandermonde
    solves over the complete basis of each field (independent of the oracle's formulas)."""
    x, y = sp.symbols("x y", real=True)
    if etype == BAR3:
        nodes_u = [(0,), (a_len,), (sp.Rational(1, 2) * a_len,)]
        basis_u = [1, x, x ** 2]
        nodes_e, basis_e = nodes_u[:2], [1, x]
        var = (x,)
    else:
        A, B = a_len, b_len
        nodes_u = [(0, 0), (A, 0), (A, B), (0, B), (A / 2, 0), (A, B / 2), (A / 2, B), (0, B / 2)]
        basis_u = [1, x, y, x ** 2, x * y, y ** 2, x ** 2 * y, x * y ** 2]
        nodes_e, basis_e = nodes_u[:4], [1, x, y, x * y]
        var = (x, y)

    def lagr(nodes, basis):
        V = sp.Matrix([[sp.sympify(f).subs(dict(zip(var, nd))) for f in basis] for nd in nodes])
        C = V.inv()
        row = sp.Matrix([basis])
        return [sp.expand((row * C[:, i])[0]) for i in range(len(nodes))]

    return var, lagr(nodes_u, basis_u), lagr(nodes_e, basis_e), nodes_u


def _sym_element(etype, m, a_len, b_len, u_coef, e_nodal):
    """Exact K, F (local dof order) of one undamaged element for a u field given as a
    polynomial and nodal ebar values; undamaged => D = 0, g = 1, dD = 0 (ebar < kappa0)."""
    var, Nu, Ne, nodes = _sym_shapes(etype, a_len, b_len)
    dim = len(var)
    E, nu, h, hs, c, t = (sp.nsimplify(getattr(m, k)) for k in ("E", "nu", "h", "h_sigma", "c", "t"))
    dom = [(v, 0, L) for v, L in zip(var, (a_len, b_len)[:dim])]
    integ = lambda f: sp.integrate(sp.expand(f), *dom)          # noqa: E731
    nd = oracle.mixed_family(etype)[5]
    nenu, nene = len(Nu), len(Ne)
    u = [sp.sympify(f) for f in u_coef]
    ebar = sum(Ne[a] * sp.nsimplify(e_nodal[a]) for a in range(nene))
    if dim == 1:
        eps = [sp.diff(u[0], var[0])]
        Cm = sp.Matrix([[E]])
        eeq, dv = eps[0], [1]                                       # reading R-1D
        B = lambda a: [[sp.diff(Nu[a], var[0])]]                    # noqa: E731
    else:
        xv, yv = var
        eps = [sp.diff(u[0], xv), sp.diff(u[1], yv), sp.diff(u[0], yv) + sp.diff(u[1], xv)]
        lam = E * nu / ((1 + nu) * (1 - 2 * nu))
        mu = E / (2 * (1 + nu))
        Cm = sp.Matrix([[lam + 2 * mu, lam, 0], [lam, lam + 2 * mu, 0], [0, 0, mu]])
        B = lambda a: [[sp.diff(Nu[a], xv), 0], [0, sp.diff(Nu[a], yv)],   # noqa: E731
                       [sp.diff(Nu[a], yv), sp.diff(Nu[a], xv)]]
        assert hs == 0            # 2D: eeq is not polynomial unless the strain is constant
        ev = [float(e) for e in eps]
        eq, d_, H_ = oracle.eqstrain(m, 2, np.array(ev))
        eeq, dv = sp.Float(eq, 30), [sp.Float(v, 30) for v in d_]
    nv = len(eps)
    sig = [sum(Cm[i, j] * eps[j] for j in range(nv)) + hs * (eeq - ebar) * dv[i] for i in range(nv)]
    K = sp.zeros(nd, nd)
    F = sp.zeros(nd, 1)
    X = Cm + hs * sp.Matrix(nv, nv, lambda i, j: dv[i] * dv[j])   # H = 0 (1D) / hs = 0 (2D)
    gradNe = [[sp.diff(Ne[a], v) for v in var] for a in range(nene)]
    gradeb = [sp.diff(ebar, v) for v in var]
    for a in range(nenu):
        Ba = sp.Matrix(B(a))
        ra = ldof(etype, a)
        fu = -t * Ba.T * sp.Matrix(sig)
        for i in range(dim):
            F[ra + i] = integ(fu[i])
        for b in range(nenu):
            Bb = sp.Matrix(B(b))
            kab = Ba.T * X * Bb
            for i in range(dim):
                for j in range(dim):
                    K[ra + i, ldof(etype, b) + j] = integ(t * kab[i, j])
        for b in range(nene):                         # 11b: -Bu^T (hs d) N_e  (dD = 0)
            kue = -(Ba.T * sp.Matrix([hs * dv[i] for i in range(nv)])) * Ne[b]
            for i in range(dim):
                K[ra + i, ldof(etype, b) + dim] = integ(t * kue[i])
    for a in range(nene):
        ra = ldof(etype, a) + dim
        F[ra] = integ(t * (Ne[a] * h * (eeq - ebar) - h * c * sum(gradNe[a][k] * gradeb[k] for k in range(dim))))
        for b in range(nenu):                         # 11c: -N_e h d^T Bu
            keu = -Ne[a] * h * (sp.Matrix([dv]) * sp.Matrix(B(b)))
            for j in range(dim):
                K[ra, ldof(etype, b) + j] = integ(t * keu[j])
        for b in range(nene):                         # 11d with g = 1, g' = 0
            K[ra, ldof(etype, b) + dim] = integ(t * (h * Ne[a] * Ne[b] + h * c * sum(
                gradNe[a][k] * gradNe[b][k] for k in range(dim))))
    return np.array(K.evalf(30), dtype=np.float64), np.array(F.evalf(30), dtype=np.float64).ravel(), nodes


@pytest.mark.parametrize("etype", [BAR3, QUAD8])
def test_element_exact_undamaged(etype):
    """whole element K, F against exact integration; rectangle a != b catches transpositions"""
    a_len, b_len = sp.Rational(5, 2), sp.Rational(3, 2)
    x, y = sp.symbols("x y", real=True)
    if etype == BAR3:
        m = mat()                                            # full R1 reading, h_sigma = h
        u_coef = [sp.Rational(3, 100000) * x + sp.Rational(2, 100000) * x ** 2]   # linear strain
        e_nodal = [3e-5, 6e-5]
    else:
        m = mat(h_sigma=0.0)                                 # 2D: constant strain, R2 reading
        u_coef = [sp.Rational(4, 100000) * x + sp.Rational(1, 100000) * y,
                  sp.Rational(-1, 100000) * x + sp.Rational(2, 100000) * y]
        e_nodal = [2e-5, 5e-5, 7e-5, 4e-5]
    Kx, Fx, nodes = _sym_element(etype, m, a_len, b_len, u_coef, e_nodal)
    dim, nenu, nene, nv, ngp, nd = oracle.mixed_family(etype)
    var = (x,) if dim == 1 else (x, y)
    Xe = np.array([[float(v) for v in nd_] for nd_ in nodes])
    Ue = np.zeros(nd)
    for a in range(nenu):
        for i in range(dim):
            Ue[ldof(etype, a) + i] = float(u_coef[i].subs(dict(zip(var, nodes[a]))))
        if a < nene:
            Ue[ldof(etype, a) + dim] = e_nodal[a]
    Ke, Fe, _, _ = oracle.mixed_element(etype, m, Xe, Ue, np.zeros(ngp))
    np.testing.assert_allclose(Ke, Kx, rtol=0, atol=1e-12 * np.abs(Kx).max())
    np.testing.assert_allclose(Fe, Fx, rtol=0, atol=1e-12 * np.abs(Fx).max())


def test_bar3_damaged_constant_state():
    """u linear, ebar constant, damaged history: every GP has the same state, so
    Fe_e = h (eps - ebar) A Le / 2 per end node and Fu = (+sigma, -sigma, 0) A with
    sigma = (1-D) E eps + h_sigma (eps - ebar) (Eq. 2; reading R-1D eeq = eps)."""
    m = mat()
    Le, eps, eb, kh = 2.0, 3e-4, 2.5e-4, 2.8e-4
    Xe = np.array([[1.0], [1.0 + Le], [1.0 + Le / 2]])
    u = lambda xx: eps * xx                                  # noqa: E731
    Ue = np.array([u(1.0), eb, u(1.0 + Le), eb, u(1.0 + Le / 2)])
    Ke, Fe, _, sig = oracle.mixed_element(BAR3, m, Xe, Ue, np.full(3, kh))
    D, _ = oracle.damage(m, kh)                              # ebar < kh: history governs
    s = (1.0 - D) * MAT["E"] * eps + MAT["h_sigma"] * (eps - eb)
    np.testing.assert_allclose(sig.ravel(), s, rtol=1e-13)
    hA = MAT["h"] * MAT["t"]
    np.testing.assert_allclose(Fe[[1, 3]], hA * (eps - eb) * Le / 2, rtol=1e-12)
    np.testing.assert_allclose(Fe[[0, 2, 4]], np.array([s, -s, 0.0]) * MAT["t"], rtol=0,
                               atol=1e-12 * abs(s))


def test_quad8_ebar_blocks_equal_q4():
    """constant strain and constant ebar (damaged): the ebar-ebar block and the ebar residual
    of a QUAD8 equal those of the Q4 oracle on the same parallelogram (both quadratures are
    exact there)"""
    m = mat()
    rng = np.random.default_rng(5)
    Xc = np.array([[0.0, 0.0], [2.0, 0.3], [2.4, 1.9], [0.4, 1.6]])   # parallelogram:
    Xm = 0.5 * (Xc + np.roll(Xc, -1, axis=0))                 # constant J, polynomial integrands
    Xe = np.vstack([Xc, Xm])
    G = np.array([[1.5e-4, 0.4e-4], [-0.2e-4, 2.5e-4]])
    uf = lambda p: G @ p                                      # noqa: E731
    eb, kh = 2.2e-4, 3.0e-4
    Uq8 = np.zeros(20)
    for a in range(8):
        Uq8[ldof(QUAD8, a):ldof(QUAD8, a) + 2] = uf(Xe[a])
        if a < 4:
            Uq8[ldof(QUAD8, a) + 2] = eb
    Uq4 = np.zeros(12)
    for a in range(4):
        Uq4[3 * a:3 * a + 2] = uf(Xc[a])
        Uq4[3 * a + 2] = eb
    K8, F8, _, s8 = oracle.mixed_element(QUAD8, m, Xe, Uq8, np.full(9, kh))
    K4, F4 = _q4(m, Xc, Uq4, kh)
    e8 = [ldof(QUAD8, a) + 2 for a in range(4)]
    e4 = [3 * a + 2 for a in range(4)]
    np.testing.assert_allclose(K8[np.ix_(e8, e8)], K4[np.ix_(e4, e4)], rtol=1e-12,
                               atol=1e-13 * np.abs(K4).max())
    np.testing.assert_allclose(F8[e8], F4[e4], rtol=1e-12, atol=1e-13 * np.abs(F4).max())
    assert np.ptp(s8, axis=0).max() <= 1e-12 * np.abs(s8).max()   # constant stress


def _q4(m, X, U, kh):
    r = oracle.element(2, m, X, U, np.full(4, kh))
    return r[0], r[1]


def _q8_patch(nx, ny, distort, seed):
    mesh = synth.mixed_mesh(QUAD8, (nx, ny), 10.0 * nx / 4)
    X = mesh.coords.copy()
    h = 10.0 / 4
    corner_ids = np.nonzero(mesh.corner)[0]
    lo, hi = X.min(axis=0), X.max(axis=0)
    rng = np.random.default_rng(seed)
    inner = np.all((X[corner_ids] > lo + 1e-9) & (X[corner_ids] < hi - 1e-9), axis=1)
    X[corner_ids[inner]] += rng.uniform(-1, 1, size=(inner.sum(), 2)) * distort * h
    for e in range(mesh.conn.shape[0]):                      # midside nodes at edge midpoints
        c = mesh.conn[e]
        for k in range(4):
            X[c[4 + k]] = 0.5 * (X[c[k]] + X[c[(k + 1) % 4]])
    return mesh, X


@pytest.mark.parametrize("kh", [0.0, 3e-4])
def test_quad8_patch(kh):
    """linear u, constant ebar on a distorted QUAD8 patch: interior u-residuals vanish,
    the stress is uniform, and sum of the ebar residuals = h (eeq - ebar) area"""
    m = mat()
    mesh, X = _q8_patch(4, 3, 0.2, 11)
    doff = oracle.mixed_dofs(QUAD8, X.shape[0], mesh.conn)
    kind = oracle.dof_kind(doff, 2)
    G = np.array([[1.2e-4, 0.3e-4], [0.5e-4, 2.0e-4]])
    eb = 1.5e-4
    dofs = np.zeros(doff[-1])
    for n in range(X.shape[0]):
        dofs[doff[n]:doff[n] + 2] = G @ X[n]
        if doff[n + 1] - doff[n] == 3:
            dofs[doff[n] + 2] = eb
    ne = mesh.conn.shape[0]
    res = oracle.mixed_assemble(QUAD8, m, X, mesh.conn, dofs, np.full((ne, 9), kh))
    lo, hi = X.min(axis=0), X.max(axis=0)
    interior = np.all((X > lo + 1e-9) & (X < hi - 1e-9), axis=1)
    rows = [doff[n] + i for n in np.nonzero(interior)[0] for i in range(2)]
    R = res["R"]
    assert np.abs(R[rows]).max() <= 1e-12 * np.abs(R).max()
    ev = np.array([G[0, 0], G[1, 1], G[0, 1] + G[1, 0]])
    eeq = oracle.eqstrain(m, 2, ev)[0]
    area = 0.0
    for c in mesh.conn[:, :4]:
        P = X[c]
        area += 0.5 * abs(np.dot(P[:, 0], np.roll(P[:, 1], -1)) - np.dot(P[:, 1], np.roll(P[:, 0], -1)))
    assert R[kind == 2].sum() == pytest.approx(MAT["h"] * (eeq - eb) * area, rel=1e-11)


# ---------------- null space, symmetry, finite differences ----------------

@pytest.mark.parametrize("etype,n", [(BAR3, (5,)), (QUAD8, (3, 2))])
def test_rigid_body_symmetry_nullity(etype, n):
    dim = oracle.mixed_family(etype)[0]
    mesh = synth.mixed_mesh(etype, n, 10.0)
    X = mesh.coords
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    kind = oracle.dof_kind(doff, dim)
    dofs, kap = synth.mixed_fields(mesh)
    res = oracle.mixed_assemble(etype, mat(), X, mesh.conn, dofs, kap)
    K = dense(res, doff[-1])
    u = kind < dim
    Kuu = K[np.ix_(u, u)]
    np.testing.assert_allclose(Kuu, Kuu.T, rtol=0, atol=1e-11 * np.abs(Kuu).max())
    node_of = np.repeat(np.arange(X.shape[0]), np.diff(doff))[u]
    comp = kind[u]
    modes = [(comp == k).astype(float) for k in range(dim)]
    if dim == 2:
        modes.append(np.where(comp == 0, -X[node_of, 1], X[node_of, 0]))
    for v in modes:
        assert np.abs(Kuu @ v).max() <= 1e-10 * np.abs(Kuu).max() * np.abs(v).max()
    # undamaged, zero strain: exactly d(d+1)/2 zero eigenvalues of Kuu (full 3-point rules)
    ne = mesh.conn.shape[0]
    res0 = oracle.mixed_assemble(etype, mat(), X, mesh.conn, np.zeros(doff[-1]), np.zeros((ne, 3 ** dim)))
    K0 = dense(res0, doff[-1])[np.ix_(u, u)]
    ev = np.linalg.eigvalsh(K0)
    nz = int((np.abs(ev) < 1e-9 * np.abs(ev).max()).sum())
    assert nz == dim * (dim + 1) // 2


@pytest.mark.parametrize("etype,n", [(BAR3, (6,)), (QUAD8, (3, 3))])
@pytest.mark.parametrize("hs", [30000.0, 0.0])
def test_tangent_finite_difference(etype, n, hs):
    dim, nenu, nene, nv, ngp, nd = oracle.mixed_family(etype)
    mesh = synth.mixed_mesh(etype, n, 10.0)
    X = mesh.coords if etype == BAR3 else _q8_patch(n[0], n[1], 0.15, 4)[1]
    dofs, _ = synth.mixed_fields(mesh)
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    kind = oracle.dof_kind(doff, dim)
    # history 2e-5 away from ebar at each GP (loading or unloading at random): no switch
    xi, _ = oracle.mixed_gauss(etype)
    Ng = np.array([oracle.mixed_shape(etype, xi[g], "e")[0] for g in range(ngp)])
    eb_nodes = np.array([[dofs[doff[c] + dim] for c in row[:nene]] for row in mesh.conn])
    ebar_gp = eb_nodes @ Ng.T
    rng = np.random.default_rng(23 + etype)
    kap = ebar_gp + np.where(rng.uniform(size=ebar_gp.shape) < 0.5, -1.0, 1.0) * 2e-5
    assert kap.min() > MAT["kappa0"] + 1e-5
    m = mat(h_sigma=hs)
    res = oracle.mixed_assemble(etype, m, X, mesh.conn, dofs, kap)
    K = dense(res, doff[-1])
    scale = np.where(kind == dim, np.abs(dofs[kind == dim]).max(), np.abs(dofs[kind < dim]).max())
    for _ in range(12):      # O(d^2) truncation: 1.2e-6 at d = 1e-4, 1.2e-8 at d = 1e-5
        v = rng.normal(size=dofs.shape) * scale
        d = 1e-5
        Rp = oracle.mixed_assemble(etype, m, X, mesh.conn, dofs + d * v, kap)["R"]
        Rm = oracle.mixed_assemble(etype, m, X, mesh.conn, dofs - d * v, kap)["R"]
        Kv = K @ v
        assert np.linalg.norm(Kv + (Rp - Rm) / (2 * d)) <= 1e-7 * np.linalg.norm(Kv)


# ---------------- dof map, pattern, assembly, history ----------------

def test_dof_map():
    mesh = synth.mixed_mesh(BAR3, (4,), 10.0)
    doff = oracle.mixed_dofs(BAR3, 9, mesh.conn)            # SPEC: 9 u-nodes, 5 ebar nodes
    assert doff[-1] == 9 + 5
    mesh = synth.mixed_mesh(QUAD8, (1, 1), 10.0)            # SPEC: 8 u-nodes, 4 ebar nodes
    doff = oracle.mixed_dofs(QUAD8, 8, mesh.conn)
    assert doff[-1] == 2 * 8 + 4
    mesh = synth.mixed_mesh(QUAD8, (3, 2), 10.0)
    assert mesh.coords.shape[0] == 7 * 5 - 3 * 2
    doff = oracle.mixed_dofs(QUAD8, mesh.coords.shape[0], mesh.conn)
    assert doff[-1] == 2 * mesh.coords.shape[0] + 4 * 3
    bad = mesh.conn.copy()
    bad[0, [1, 4]] = bad[0, [4, 1]]          # a corner shared with element 1 used as a midside node
    with pytest.raises(ValueError):
        oracle.mixed_dofs(QUAD8, mesh.coords.shape[0], bad)


@pytest.mark.parametrize("etype,n", [(BAR3, (5,)), (QUAD8, (3, 2))])
def test_pattern_and_assembly_brute_force(etype, n):
    dim, nenu, nene, nv, ngp, nd = oracle.mixed_family(etype)
    mesh = synth.mixed_mesh(etype, n, 10.0)
    X = mesh.coords
    dofs, kap = synth.mixed_fields(mesh)
    doff = oracle.mixed_dofs(etype, X.shape[0], mesh.conn)
    nn = X.shape[0]
    m = mat()
    Kd = np.zeros((doff[-1], doff[-1]))
    Rd = np.zeros(doff[-1])
    nodes_adj = set()
    for e, c in enumerate(mesh.conn):
        g = np.concatenate([doff[c[a]] + np.arange(dim + 1 if a < nene else dim) for a in range(nenu)])
        Ke, Fe, _, _ = oracle.mixed_element(etype, m, X[c], dofs[g], kap[e])
        np.add.at(Kd, (g[:, None], g[None, :]), Ke)
        np.add.at(Rd, g, Fe)
        nodes_adj |= {(a, b) for a in c for b in c}
    res = oracle.mixed_assemble(etype, m, X, mesh.conn, dofs, kap)
    Kp = dense(res, doff[-1])
    np.testing.assert_allclose(Kp, Kd, rtol=1e-14, atol=1e-14 * np.abs(Kd).max())
    np.testing.assert_allclose(res["R"], Rd, rtol=1e-14, atol=1e-14 * np.abs(Rd).max())
    # pattern = all dof pairs of node pairs sharing an element, ascending columns
    want = sum((doff[a + 1] - doff[a]) * (doff[b + 1] - doff[b]) for a, b in nodes_adj)
    assert res["col_idx"].size == want
    rp, ci = res["row_ptr"], res["col_idx"]
    for r in range(doff[-1]):
        assert np.all(np.diff(ci[rp[r]:rp[r + 1]]) > 0)
    assert nn == X.shape[0]


@pytest.mark.parametrize("etype", [BAR3, QUAD8])
def test_update_history(etype):
    dim, nenu, nene, nv, ngp, nd = oracle.mixed_family(etype)
    mesh = synth.mixed_mesh(etype, (4,) if etype == BAR3 else (3, 2), 10.0)
    dofs, kap = synth.mixed_fields(mesh)
    doff = oracle.mixed_dofs(etype, mesh.coords.shape[0], mesh.conn)
    k1 = oracle.mixed_update_history(etype, mesh.conn, doff, dofs, kap)
    # brute force: ebar at the physical Gauss points by linear / bilinear interpolation
    p = np.sqrt(0.6)
    pts = [-p, 0.0, p]
    for e, c in enumerate(mesh.conn):
        ebn = np.array([dofs[doff[c[a]] + dim] for a in range(nene)])
        for g in range(ngp):
            s = pts[g % 3]
            if dim == 1:
                eb = 0.5 * (1 - s) * ebn[0] + 0.5 * (1 + s) * ebn[1]
            else:
                t = pts[g // 3]
                eb = 0.25 * ((1 - s) * (1 - t) * ebn[0] + (1 + s) * (1 - t) * ebn[1] +
                             (1 + s) * (1 + t) * ebn[2] + (1 - s) * (1 + t) * ebn[3])
            want = eb if eb - kap[e, g] > 1e-10 else kap[e, g]
            assert k1[e, g] == pytest.approx(want, rel=1e-14)
    assert np.all(k1 >= kap)


# ---------------- state update (Alg. 2 l.8-14) for mixed elements ----------------

def test_bar3_state_closed_form():
    """u = a x + b x^2 on a BAR3 mesh: eps at the physical Gauss points = a + 2 b x_g exactly
    (the quadratic field is reproduced); eeq = eps (R-1D), d = 1; kappa by the history rule;
    D, g from Eqs. A.1, A.4; sigma of Eq. 2."""
    m = mat()
    n = 6
    mesh = synth.mixed_mesh(BAR3, (n,), 12.0)
    X = mesh.coords
    doff = oracle.mixed_dofs(BAR3, X.shape[0], mesh.conn)
    a, b = 1e-4, 2e-5
    dofs = np.zeros(doff[-1])
    for k in range(X.shape[0]):
        dofs[doff[k]] = a * X[k, 0] + b * X[k, 0] ** 2
        if doff[k + 1] - doff[k] == 2:
            dofs[doff[k] + 1] = 1.5e-4 + 1e-5 * X[k, 0]
    kap0 = np.full((n, 3), 2.0e-4)
    sdv, k1 = oracle.mixed_update_state(BAR3, m, X, mesh.conn, doff, dofs, kap0)
    pts = np.array([-np.sqrt(0.6), 0.0, np.sqrt(0.6)])
    for e, c in enumerate(mesh.conn):
        x0, x1 = X[c[0], 0], X[c[1], 0]
        for g in range(3):
            xg = 0.5 * (x0 + x1) + 0.5 * (x1 - x0) * pts[g]
            eps = a + 2 * b * xg
            eb = 1.5e-4 + 1e-5 * xg
            kap = eb if eb - kap0[e, g] > 1e-10 else kap0[e, g]
            D, _ = oracle.damage(m, kap)
            gI, _ = oracle.interaction(m, D)
            want = [eps, 1.0, (1 - D) * MAT["E"] * eps + MAT["h_sigma"] * (eps - eb), eps, eb,
                    kap, D, gI]
            np.testing.assert_allclose(sdv[e, g], want, rtol=1e-12, atol=1e-20)
    np.testing.assert_array_equal(k1, sdv[:, :, 5])


def test_quad8_state_patch_and_consistency():
    """linear u on a distorted QUAD8 patch: uniform strain, sigma = C eps (plane strain,
    textbook Lame constants) while undamaged; the records' sigma equals the stress the element
    routine reports at every GP"""
    m = mat()
    mesh, X = _q8_patch(3, 2, 0.2, 7)
    doff = oracle.mixed_dofs(QUAD8, X.shape[0], mesh.conn)
    G = np.array([[2e-5, 1e-5], [-0.5e-5, 3e-5]])
    dofs = np.zeros(doff[-1])
    for k in range(X.shape[0]):
        dofs[doff[k]:doff[k] + 2] = G @ X[k]
        if doff[k + 1] - doff[k] == 3:
            dofs[doff[k] + 2] = 5e-5
    ne = mesh.conn.shape[0]
    sdv, _ = oracle.mixed_update_state(QUAD8, m, X, mesh.conn, doff, dofs, np.zeros((ne, 9)))
    ev = np.array([G[0, 0], G[1, 1], G[0, 1] + G[1, 0]])
    E, nu = MAT["E"], MAT["nu"]
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    eeq, dv, _ = oracle.eqstrain(m, 2, ev)
    sig = np.array([(lam + 2 * mu) * ev[0] + lam * ev[1], lam * ev[0] + (lam + 2 * mu) * ev[1],
                    mu * ev[2]]) + MAT["h_sigma"] * (eeq - 5e-5) * dv
    for e in range(ne):
        np.testing.assert_allclose(sdv[e, :, 0:3], np.tile(ev, (9, 1)), rtol=1e-11, atol=1e-18)
        np.testing.assert_allclose(sdv[e, :, 6:9], np.tile(sig, (9, 1)), rtol=1e-10)
        np.testing.assert_allclose(sdv[e, :, 12], 0.0, atol=0)            # D = 0
        g = mesh.conn[e]
        gd = np.concatenate([doff[g[a]] + np.arange(3 if a < 4 else 2) for a in range(8)])
        _, _, _, s_el = oracle.mixed_element(QUAD8, m, X[g], dofs[gd], np.zeros(9))
        np.testing.assert_allclose(sdv[e, :, 6:9], s_el, rtol=1e-13, atol=1e-13 * np.abs(s_el).max())


def test_bar3_ebar_blocks_equal_bar2():
    """constant strain and constant ebar (damaged): the ebar-ebar block and the ebar residual
    of a BAR3 equal those of the (separately pinned) BAR2 oracle on the same end nodes"""
    m = mat()
    x0, x1, eps, eb, kh = 1.5, 3.7, 2.5e-4, 2.2e-4, 3.0e-4
    Xe = np.array([[x0], [x1], [0.5 * (x0 + x1)]])
    u = lambda x: eps * x                                   # noqa: E731
    U3 = np.array([u(x0), eb, u(x1), eb, u(0.5 * (x0 + x1))])
    U2 = np.array([u(x0), eb, u(x1), eb])
    K3, F3, _, _ = oracle.mixed_element(BAR3, m, Xe, U3, np.full(3, kh))
    r = oracle.element(1, m, np.array([[x0], [x1]]), U2, np.full(2, kh))
    K2, F2 = r[0], r[1]
    e3, e2 = [1, 3], [1, 3]
    np.testing.assert_allclose(K3[np.ix_(e3, e3)], K2[np.ix_(e2, e2)], rtol=1e-12,
                               atol=1e-13 * np.abs(K2).max())
    np.testing.assert_allclose(F3[e3], F2[e2], rtol=1e-12, atol=1e-13 * np.abs(F2).max())


def test_r_rel_precision_pin():
    """Reading R-REL: the oracle (and every kernel) evaluates J and the
    gradients on coordinates relative to the element's node 0.  Pin: for a QUAD8 element of
    the bench mesh's size (h = 0.2 mm) at the far corner of the 100 mm plate, the undamaged
    elastic Kuu (h_sigma = 0, D = 0: the textbook integral of B^T C B over the element) is
    evaluated exactly with mpmath at 50 digits.  A plain FP64 evaluation on ABSOLUTE
    coordinates is off by ~|X| / h x eps (cancellation in J = sum_a X_a dN_a/dxi); the same
    FP64 evaluation on RELATIVE coordinates, and the oracle, are within a few eps of the
    exact value."""
    import mpmath as mp
    mp.mp.dps = 50
    h, x0, y0 = 0.2, 99.8, 99.6
    # straight-edged, distorted quadrilateral; midside nodes at the edge midpoints (R-GEO)
    cor = [(0.0, 0.0), (h, 0.013), (h + 0.021, h - 0.007), (-0.017, h)]
    mids = [tuple((cor[i][k] + cor[(i + 1) % 4][k]) / 2 for k in range(2)) for i in range(4)]
    rel = cor + mids
    xi_n = [(-1, -1), (1, -1), (1, 1), (-1, 1), (0, -1), (1, 0), (0, 1), (-1, 0)]

    def dshape(xi, eta, one):
        """dN/dxi, dN/deta of the serendipity QUAD8 at (xi, eta) in the number type of `one`"""
        out = []
        for (a, b) in xi_n:
            if a != 0 and b != 0:
                dx = one * a * (1 + b * eta) * (2 * a * xi + b * eta) / 4
                dy = one * b * (1 + a * xi) * (a * xi + 2 * b * eta) / 4
            elif a == 0:
                dx = -xi * (1 + b * eta) * one
                dy = one * b * (1 - xi * xi) / 2
            else:
                dx = one * a * (1 - eta * eta) / 2
                dy = -eta * (1 + a * xi) * one
            out.append((dx, dy))
        return out

    E, nu = 30000.0, 0.2

    def kuu(X, num, sqrt35, w):
        lam = num(E) * num(nu) / ((1 + num(nu)) * (1 - 2 * num(nu)))
        mu = num(E) / (2 * (1 + num(nu)))
        K = [[num(0)] * 16 for _ in range(16)]
        gp = [-sqrt35, num(0), sqrt35]
        for j, eta in enumerate(gp):
            for i, xi in enumerate(gp):
                dN = dshape(xi, eta, num(1))
                J = [[sum(X[a][r] * dN[a][c] for a in range(8)) for c in range(2)] for r in range(2)]
                det = J[0][0] * J[1][1] - J[0][1] * J[1][0]
                gx = [(J[1][1] * d[0] - J[1][0] * d[1]) / det for d in dN]
                gy = [(-J[0][1] * d[0] + J[0][0] * d[1]) / det for d in dN]
                wd = w[i] * w[j] * det
                for a in range(8):
                    for b in range(8):
                        K[2 * a][2 * b] += wd * ((lam + 2 * mu) * gx[a] * gx[b] + mu * gy[a] * gy[b])
                        K[2 * a][2 * b + 1] += wd * (lam * gx[a] * gy[b] + mu * gy[a] * gx[b])
                        K[2 * a + 1][2 * b] += wd * (lam * gy[a] * gx[b] + mu * gx[a] * gy[b])
                        K[2 * a + 1][2 * b + 1] += wd * ((lam + 2 * mu) * gy[a] * gy[b] + mu * gx[a] * gx[b])
        return K

    absX = [(x0 + p[0], y0 + p[1]) for p in rel]
    Xmp = [(mp.mpf(a), mp.mpf(b)) for a, b in absX]   # the mesh's FP64 coordinates, exactly
    exact = kuu([(a - Xmp[0][0], b - Xmp[0][1]) for a, b in Xmp], mp.mpf, mp.sqrt(mp.mpf(3) / 5),
                [mp.mpf(5) / 9, mp.mpf(8) / 9, mp.mpf(5) / 9])
    f64 = lambda v: np.float64(v)
    s35, w64 = np.sqrt(0.6), [5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0]
    k_abs = kuu(absX, f64, s35, w64)
    k_rel = kuu([(a - absX[0][0], b - absX[0][1]) for a, b in absX], f64, s35, w64)
    # the oracle on the same element (absolute coordinates in, R-REL inside), undamaged
    mat = oracle.material(**dict(synth.MATERIAL, h_sigma=0.0))
    Xe = np.array(absX)
    Ue = np.zeros(20)
    Ke, _, _, _ = oracle.mixed_element(synth.QUAD8, mat, Xe, Ue, np.full(9, synth.MATERIAL["kappa0"]))
    udof = [a * 3 + i if a < 4 else 12 + (a - 4) * 2 + i for a in range(8) for i in range(2)]
    k_orc = Ke[np.ix_(udof, udof)]

    ex = np.array([[float(v) for v in row] for row in exact])
    rowmax = np.abs(ex).max(axis=1)[:, None]
    e_abs = (np.abs(np.array(k_abs) - ex) / rowmax).max()
    e_rel = (np.abs(np.array(k_rel) - ex) / rowmax).max()
    e_orc = (np.abs(k_orc - ex) / rowmax).max()
    print(f"R-REL pin: absolute {e_abs:.2e}, relative {e_rel:.2e}, oracle {e_orc:.2e} (x row max)")
    assert e_rel < 2e-15 and e_orc < 2e-15
    assert e_abs > 20 * max(e_rel, e_orc) and e_abs > 1e-14
