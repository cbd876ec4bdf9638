"""Pins of the oracle's state-variable update (Alg. 2 l.8-14, Fig. 9a
`update_variables`, P:288-295 / P:359-390) and of the per-GP defect fields -- CPU.

Pinned against: SURVEY Appendix A values (tests/golden/appendix_a.json), fields that bilinear /
trilinear elements reproduce exactly (homogeneous strain, pure shear -> reading R-SH),
closed-form elasticity in the undamaged regime, the alpha = 0 and kappa < kappa0 special cases
of Eq. A.1, central differences of eeq (Alg. 2 l.11), and the history rule of Fig. 9a l.22-24.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))
MAT = dict(E=30000.0, nu=0.2, k=10.0, kappa0=1e-4, alpha=0.99, beta=300.0, h=30000.0,
           h_sigma=30000.0, c=2.0, R=0.05, n=5.0, t=1.0)


def m(**kw):
    d = dict(MAT)
    d.update(kw)
    return oracle.material(**d)


def unit_element(etype):
    """one element on the unit interval / square / cube, nodes in the reference order"""
    ref = {oracle.BAR2: [[0.0], [1.0]],
           oracle.QUAD4: [[0, 0], [1, 0], [1, 1], [0, 1]],
           oracle.HEX8: [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                         [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]]}[etype]
    X = np.array(ref, dtype=np.float64)
    return X, np.arange(X.shape[0], dtype=np.int64)[None, :]


def dofs_from(etype, X, u_fn, ebar):
    dim, nen, ndpn = oracle.FAMILY[etype][:3]
    d = np.zeros((X.shape[0], ndpn))
    for a in range(X.shape[0]):
        d[a, :dim] = u_fn(X[a])
        d[a, dim] = ebar
    return d.reshape(-1)


def split(etype, rec):
    nv = oracle.FAMILY[etype][3]
    return dict(eps=rec[:nv], d=rec[nv:2 * nv], sig=rec[2 * nv:3 * nv], eeq=rec[3 * nv],
                ebar=rec[3 * nv + 1], kappa=rec[3 * nv + 2], D=rec[3 * nv + 3], g=rec[3 * nv + 4])


def test_width():
    assert [oracle.sdv_width(t) for t in (1, 2, 3)] == [8, 14, 23]


@pytest.mark.parametrize("kappa,D,dD", GOLD["damage"])
def test_bar_damage_golden(kappa, D, dD):
    """1D bar, uniform strain eps, ebar = kappa > kappa_hist: D(kappa) is Appendix A's value,
    sigma = (1 - D) E eps + h_sigma (eeq - ebar) (Eq. 2, eeq = eps by reading R-1D)."""
    X, conn = unit_element(oracle.BAR2)
    eps = 3e-4
    d = dofs_from(oracle.BAR2, X, lambda x: [eps * x[0]], kappa)
    kh = np.full(2, 0.5e-4)
    sdv, kn = oracle.update_state(oracle.BAR2, m(), X, conn, d, kh)
    for g in range(2):
        r = split(oracle.BAR2, sdv[0, g])
        assert r["eps"][0] == pytest.approx(eps, rel=1e-14)
        assert r["eeq"] == pytest.approx(eps, rel=1e-14)
        assert r["ebar"] == pytest.approx(kappa, rel=1e-14)
        loading = kappa - 0.5e-4 > 1e-10
        assert r["kappa"] == pytest.approx(kappa if loading else 0.5e-4, rel=1e-15)
        Dexp = D if loading else 0.0
        assert r["D"] == pytest.approx(Dexp, rel=1e-13, abs=1e-300)
        assert r["sig"][0] == pytest.approx((1 - Dexp) * MAT["E"] * eps +
                                            MAT["h_sigma"] * (eps - kappa), rel=1e-12)
        assert r["d"][0] == 1.0
    assert np.all(kn == sdv[0, :, 3 * 1 + 2])


@pytest.mark.parametrize("D,g,dg", GOLD["interaction"])
def test_interaction_at_golden_damage(D, g, dg):
    """g of the record at a state whose damage is D (alpha = 0 gives D = 1 - kappa0/kappa, so
    kappa = kappa0 / (1 - D) hits each tabulated D exactly up to rounding)"""
    if D >= 1.0:
        pytest.skip("D = 1 needs kappa -> infinity")
    X, conn = unit_element(oracle.BAR2)
    kap = MAT["kappa0"] / (1.0 - D) if D > 0 else 0.5e-4
    d = dofs_from(oracle.BAR2, X, lambda x: [0.0], kap)
    sdv, _ = oracle.update_state(oracle.BAR2, m(alpha=0.0), X, conn, d, np.full(2, 0.2e-4))
    r = split(oracle.BAR2, sdv[0, 0])
    assert r["D"] == pytest.approx(D, rel=1e-12, abs=1e-15)
    assert r["g"] == pytest.approx(g, rel=1e-11)


@pytest.mark.parametrize("etype", [oracle.QUAD4, oracle.HEX8])
def test_homogeneous_strain_and_elastic_stress(etype):
    """u = (e1 x, e2 y[, e3 z]) + shear (gamma y in u_x): bilinear / trilinear elements reproduce
    it exactly -> Voigt strain [e1, e2, (e3), gamma, 0, 0] at every GP (engineering shear, R-SH).
    Undamaged (ebar below kappa0) with h_sigma = 0: sigma = C eps, plane strain in 2D (R-PS)."""
    X, conn = unit_element(etype)
    dim = oracle.FAMILY[etype][0]
    e = [2e-5, -1e-5, 0.5e-5][:dim]
    gam = 3e-5
    def u(x):
        v = [e[i] * x[i] for i in range(dim)]
        v[0] += gam * x[1]
        return v
    d = dofs_from(etype, X, u, 0.5e-4)
    ngp = oracle.FAMILY[etype][4]
    sdv, _ = oracle.update_state(etype, m(h_sigma=0.0), X, conn, d, np.zeros(ngp))
    E, nu = MAT["E"], MAT["nu"]
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    tr = sum(e)
    for g in range(ngp):
        r = split(etype, sdv[0, g])
        if dim == 2:
            eps_exp = [e[0], e[1], gam]
            sig_exp = [lam * tr + 2 * mu * e[0], lam * tr + 2 * mu * e[1], mu * gam]
        else:
            eps_exp = [e[0], e[1], e[2], gam, 0.0, 0.0]
            sig_exp = [lam * tr + 2 * mu * e[i] for i in range(3)] + [mu * gam, 0.0, 0.0]
        np.testing.assert_allclose(r["eps"], eps_exp, rtol=1e-12, atol=1e-20)
        np.testing.assert_allclose(r["sig"], sig_exp, rtol=1e-12, atol=1e-12)
        assert r["D"] == 0.0 and r["g"] == 1.0


@pytest.mark.parametrize("etype", [oracle.QUAD4, oracle.HEX8])
def test_deeq_matches_central_differences(etype):
    """Alg. 2 l.11 output d eeq / d eps_v against central differences of the record's eeq
    (perturbing one homogeneous strain component at a time)"""
    X, conn = unit_element(etype)
    dim, nen, ndpn, nv, ngp, nd = oracle.FAMILY[etype]
    base = np.array([3e-5, -1e-5, 2e-5, 1.5e-5, -0.7e-5, 0.4e-5])[:nv]
    def rec(ev):
        # displacement reproducing the Voigt strain ev exactly (engineering shear)
        def u(x):
            if dim == 2:
                return [ev[0] * x[0] + ev[2] * x[1], ev[1] * x[1]]
            return [ev[0] * x[0] + ev[3] * x[1] + ev[5] * x[2], ev[1] * x[1] + ev[4] * x[2],
                    ev[2] * x[2]]
        s, _ = oracle.update_state(etype, m(), X, conn, dofs_from(etype, X, u, 0.0), np.zeros(ngp))
        return split(etype, s[0, 0])
    r0 = rec(base)
    np.testing.assert_allclose(r0["eps"], base, rtol=1e-12)
    h = 1e-9
    for V in range(nv):
        ep, em = base.copy(), base.copy()
        ep[V] += h
        em[V] -= h
        fd = (rec(ep)["eeq"] - rec(em)["eeq"]) / (2 * h)
        assert r0["d"][V] == pytest.approx(fd, rel=1e-5, abs=1e-7)


def test_defect_fields():
    """per-GP kappa0 / alpha: a GP with kappa0 above its kappa stays undamaged; alpha = 0
    gives D = 1 - kappa0/kappa exactly (Eq. A.1); material values reproduce the uniform run"""
    X, conn = unit_element(oracle.QUAD4)
    ngp = 4
    kap = 3e-4
    d = dofs_from(oracle.QUAD4, X, lambda x: [1e-5 * x[0], 0.0], kap)
    kh = np.zeros(ngp)
    k0 = np.array([1e-4, 5e-4, 2e-4, 1e-4])
    al = np.array([0.99, 0.99, 0.0, 0.5])
    sdv, _ = oracle.update_state(oracle.QUAD4, m(), X, conn, d, kh, kappa0_gp=k0, alpha_gp=al)
    D = [split(oracle.QUAD4, sdv[0, g])["D"] for g in range(ngp)]
    ref = {r[0]: r[1] for r in GOLD["damage"]}
    assert D[0] == pytest.approx(ref[3e-4], rel=1e-13)          # the material values
    assert D[1] == 0.0                                            # kappa < kappa0_gp
    assert D[2] == pytest.approx(1 - 2e-4 / kap, rel=1e-14)       # alpha = 0
    ex = math.exp(-MAT["beta"] * (kap - 1e-4))
    assert D[3] == pytest.approx(1 - (1e-4 / kap) * (1 - 0.5 + 0.5 * ex), rel=1e-14)
    s_uni, _ = oracle.update_state(oracle.QUAD4, m(), X, conn, d, kh)
    s_def, _ = oracle.update_state(oracle.QUAD4, m(), X, conn, d, kh,
                                   kappa0_gp=np.full(ngp, MAT["kappa0"]),
                                   alpha_gp=np.full(ngp, MAT["alpha"]))
    assert np.array_equal(s_uni, s_def)


def test_history_commit_rule():
    """Fig. 9a l.22-24: kappa <- ebar where ebar - kappa_hist > 1e-10, else kept (R-TH)"""
    X, conn = unit_element(oracle.BAR2)
    for kh0, eb, exp in ((1e-4, 2e-4, 2e-4), (2e-4, 1e-4, 2e-4), (2e-4, 2e-4 + 5e-11, 2e-4)):
        d = dofs_from(oracle.BAR2, X, lambda x: [0.0], eb)
        _, kn = oracle.update_state(oracle.BAR2, m(), X, conn, d, np.full(2, kh0))
        np.testing.assert_allclose(kn, exp, rtol=2e-16 * 4, atol=0)
