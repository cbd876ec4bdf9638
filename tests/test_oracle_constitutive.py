"""Pins of the oracle's pointwise laws (Appendix A of PAPER.md) -- CPU only.

Each test pins the oracle to something other than itself: values printed in SURVEY
Appendix A (40-digit evaluation, tests/golden/appendix_a.json), closed-form limits,
a principal-strain route to the invariants, homogeneity, and central differences.
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


# ---------------- Eq. A.1 damage law, Fig. 8b threshold ----------------

@pytest.mark.parametrize("kappa,D,dD", GOLD["damage"])
def test_damage_golden(kappa, D, dD):
    Dv, dDv = oracle.damage(m(), kappa)
    assert Dv == pytest.approx(D, rel=1e-14, abs=1e-300)
    assert dDv == pytest.approx(dD, rel=1e-13, abs=1e-300)


def test_damage_limits_and_monotone():
    mat = m()
    assert oracle.damage(mat, 0.5e-4) == (0.0, 0.0)          # kappa <= kappa0 branch (Eq. A.1)
    assert oracle.damage(mat, 1e-4)[0] == 0.0                # continuity at kappa0
    ks = np.linspace(0.5e-4, 50e-4, 1000)
    Ds = np.array([oracle.damage(mat, k)[0] for k in ks])
    assert np.all(np.diff(Ds) >= 0.0) and Ds.min() >= 0.0 and Ds.max() < 1.0
    # just above the threshold D -> 0 continuously
    assert oracle.damage(mat, 1e-4 * (1 + 1e-5))[0] < 1e-4


@pytest.mark.parametrize("kappa", [1.3e-4, 2.7e-4, 6e-4, 3e-3])
def test_damage_derivative_fd(kappa):
    mat = m()
    hstep = kappa * 1e-6
    fd = (oracle.damage(mat, kappa + hstep)[0] - oracle.damage(mat, kappa - hstep)[0]) / (2 * hstep)
    assert oracle.damage(mat, kappa)[1] == pytest.approx(fd, rel=1e-7)


def test_damage_alpha_beta_special_case():
    # alpha = 0: D = 1 - kappa0/kappa (exponential term drops) -- closed form
    mat = m(alpha=0.0)
    for k in (2e-4, 5e-4):
        assert oracle.damage(mat, k)[0] == pytest.approx(1 - 1e-4 / k, rel=1e-15)
        assert oracle.damage(mat, k)[1] == pytest.approx(1e-4 / k**2, rel=1e-15)


# ---------------- Eq. A.4 interaction function ----------------

@pytest.mark.parametrize("D,g,dg", GOLD["interaction"])
def test_interaction_golden(D, g, dg):
    gv, dgv = oracle.interaction(m(), D)
    assert gv == pytest.approx(g, rel=1e-14)
    assert dgv == pytest.approx(dg, rel=1e-14)


@pytest.mark.parametrize("R,n", [(0.05, 5.0), (0.2, 1.0), (0.01, 12.0)])
def test_interaction_limits(R, n):
    mat = m(R=R, n=n)
    assert oracle.interaction(mat, 0.0)[0] == pytest.approx(1.0, rel=1e-15)   # g(0) = 1
    assert oracle.interaction(mat, 1.0)[0] == pytest.approx(R, rel=1e-14)     # g(1) = R
    for D in (0.1, 0.5, 0.8):
        hstep = 1e-6
        fd = (oracle.interaction(mat, D + hstep)[0] - oracle.interaction(mat, D - hstep)[0]) / (2 * hstep)
        assert oracle.interaction(mat, D)[1] == pytest.approx(fd, rel=1e-8)


@pytest.mark.parametrize("kappa,gp", GOLD["gprime_of_kappa"])
def test_gprime_golden(kappa, gp):
    mat = m()
    D, dD = oracle.damage(mat, kappa)
    assert oracle.interaction(mat, D)[1] * dD == pytest.approx(gp, rel=1e-13)


# ---------------- Eq. A.3 equivalent strain, reading R-A3 ----------------

def _voigt3(eps):
    """3x3 tensor -> 3D Voigt [xx,yy,zz,gxy,gyz,gxz] (engineering shear)."""
    return np.array([eps[0, 0], eps[1, 1], eps[2, 2], 2 * eps[0, 1], 2 * eps[1, 2], 2 * eps[0, 2]])


def _principal_eeq(eps, k, nu, c3):
    """Eq. A.3 from PRINCIPAL strains (numpy eigvalsh): a route independent of the oracle's."""
    e = np.linalg.eigvalsh(eps)
    I1 = e.sum()
    J2 = ((e[0] - e[1]) ** 2 + (e[1] - e[2]) ** 2 + (e[2] - e[0]) ** 2) / 6.0
    c1 = (k - 1) / (2 * k * (1 - 2 * nu))
    c2 = ((k - 1) / (1 - 2 * nu)) ** 2
    return c1 * I1 + math.sqrt(c2 * I1 * I1 + c3 * J2) / (2 * k)


@pytest.mark.parametrize("nu", [0.0, 0.2, 0.35])
@pytest.mark.parametrize("k", [1.0, 10.0, 20.0])
def test_eqstrain_uniaxial_stress_tension_compression(nu, k):
    """k = compressive/tensile strength ratio: uniaxial stress tension eps -> eps,
    compression -eps -> eps/k.  Holds exactly for the de Vree constants only."""
    mat = m(nu=nu, k=k)
    for s in (1e-4, 3.3e-3):
        for sign, expect in ((1.0, s), (-1.0, s / k)):
            ev = np.array([sign * s, -nu * sign * s, -nu * sign * s, 0, 0, 0])
            assert oracle.eqstrain(mat, 3, ev)[0] == pytest.approx(expect, rel=1e-13)
    # the printed constants (eq_variant 1) do NOT have this property (reading R-A3)
    lit = m(nu=nu, k=k, eq_variant=1)
    if k > 1 and nu > 0:
        ev = np.array([1e-4, -nu * 1e-4, -nu * 1e-4, 0, 0, 0])
        assert abs(oracle.eqstrain(lit, 3, ev)[0] - 1e-4) > 1e-7


def test_eqstrain_golden_values():
    mat = m()
    g = GOLD["eqstrain_devree"]
    assert oracle.eqstrain(mat, 2, [0, 2e-4, 0])[0] == pytest.approx(g["plane_strain_uniaxial_eyy_2e-4"], rel=1e-14)
    assert oracle.eqstrain(mat, 2, [0, 0, 2e-4])[0] == pytest.approx(g["pure_shear_eps12_1e-4"], rel=1e-14)
    lit = m(eq_variant=1)
    g = GOLD["eqstrain_literal"]
    assert oracle.eqstrain(lit, 3, [1e-4, -2e-5, -2e-5, 0, 0, 0])[0] == pytest.approx(g["uniaxial_stress_tension_1e-4"], rel=1e-13)
    assert oracle.eqstrain(lit, 3, [-1e-4, 2e-5, 2e-5, 0, 0, 0])[0] == pytest.approx(g["uniaxial_stress_compression_-1e-4"], rel=1e-12)
    assert oracle.eqstrain(lit, 2, [0, 2e-4, 0])[0] == pytest.approx(g["plane_strain_uniaxial_eyy_2e-4"], rel=1e-14)
    assert oracle.eqstrain(lit, 2, [0, 0, 2e-4])[0] == pytest.approx(g["pure_shear_eps12_1e-4"], rel=1e-14)


def test_eqstrain_principal_route_and_plane_strain():
    """Random tensors: oracle (Voigt, dev:dev) == principal-strain evaluation; 2D plane strain
    == 3D with eps33 = eps13 = eps23 = 0 (reading R-PS)."""
    rng = np.random.default_rng(1)
    for variant, c3 in ((0, 12 * 10 / 1.2**2), (1, 2 * 10 / 0.8**2)):
        mat = m(eq_variant=variant)
        for _ in range(100):
            A = rng.normal(size=(3, 3)) * 1e-4
            eps = 0.5 * (A + A.T)
            e3 = oracle.eqstrain(mat, 3, _voigt3(eps))[0]
            assert e3 == pytest.approx(_principal_eeq(eps, 10.0, 0.2, c3), rel=1e-12)
            eps[2, :] = 0
            eps[:, 2] = 0
            e2 = oracle.eqstrain(mat, 2, [eps[0, 0], eps[1, 1], 2 * eps[0, 1]])[0]
            assert e2 == pytest.approx(_principal_eeq(eps, 10.0, 0.2, c3), rel=1e-12)


def test_eqstrain_homogeneity_and_zero():
    mat = m()
    rng = np.random.default_rng(2)
    for dim, nv in ((2, 3), (3, 6)):
        for _ in range(20):
            ev = rng.normal(size=nv) * 1e-4
            e = oracle.eqstrain(mat, dim, ev)[0]
            for lam in (2.0, 10.0, 0.5):
                assert oracle.eqstrain(mat, dim, lam * ev)[0] == pytest.approx(lam * e, rel=1e-13)
        e, d, H = oracle.eqstrain(mat, dim, np.zeros(nv))
        assert e == 0.0
        c1 = 9 / (20 * 0.6)
        mvec = np.array([1, 1, 0] if dim == 2 else [1, 1, 1, 0, 0, 0], dtype=float)
        np.testing.assert_allclose(d, c1 * mvec, rtol=1e-15)      # reading R-SQ
        assert np.all(H == 0.0)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("variant", [0, 1])
def test_eqstrain_derivatives_fd(dim, variant):
    mat = m(eq_variant=variant)
    nv = 3 if dim == 2 else 6
    rng = np.random.default_rng(3 + dim)
    for _ in range(30):
        ev = rng.normal(size=nv) * 1e-4
        e, d, H = oracle.eqstrain(mat, dim, ev)
        hstep = 1e-10
        for V in range(nv):
            ep, dp, _ = oracle.eqstrain(mat, dim, ev + hstep * np.eye(nv)[V])
            em, dm, _ = oracle.eqstrain(mat, dim, ev - hstep * np.eye(nv)[V])
            assert d[V] == pytest.approx((ep - em) / (2 * hstep), rel=1e-6, abs=1e-8)
            np.testing.assert_allclose(H[:, V], (dp - dm) / (2 * hstep), rtol=1e-5,
                                       atol=1e-5 * np.abs(H).max())
        np.testing.assert_allclose(H, H.T, rtol=1e-13, atol=1e-13 * np.abs(H).max())


def test_eqstrain_1d():
    mat = m()
    for s in (3e-4, -2e-4):
        e, d, H = oracle.eqstrain(mat, 1, [s])
        assert (e, d[0], H[0, 0]) == (s, 1.0, 0.0)                # reading R-1D
