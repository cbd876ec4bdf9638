"""Pins of the blocked DOF order [u; ebar] (`u(1:ndof_u)` then the ebar
dofs) -- CPU.  The permutation is pinned against a hand-written 1D
example; the permuted CSR against the dense P K P^T and the u-u block against the dense
restriction of K to the u dofs."""
import numpy as np
import pytest

import oracle
import synth


def _res(etype, n):
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    d, k = synth.fields(cfg, mesh)
    res = oracle.assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn, d, k)
    return mesh, res


def _dense(res, n):
    K = np.zeros((n, n))
    for r in range(n):
        for q in range(res["row_ptr"][r], res["row_ptr"][r + 1]):
            K[r, res["col_idx"][q]] = res["val"][q]
    return K


def test_perm_hand_example():
    # 1D bar, 3 nodes: interleaved [u0 e0 u1 e1 u2 e2] -> blocked [u0 u1 u2 e0 e1 e2]
    assert list(oracle.blocked_perm(oracle.BAR2, 3)) == [0, 2, 4, 1, 3, 5]
    # Q4, 2 nodes: [ux0 uy0 e0 ux1 uy1 e1] -> [ux0 uy0 ux1 uy1 e0 e1]
    assert list(oracle.blocked_perm(oracle.QUAD4, 2)) == [0, 1, 3, 4, 2, 5]


@pytest.mark.parametrize("etype,n", [(1, (5,)), (2, (3, 2)), (3, (2, 1, 2))])
def test_blocked_is_symmetric_permutation(etype, n):
    mesh, res = _res(etype, n)
    nn = mesh.coords.shape[0]
    ndpn, dim = oracle.FAMILY[etype][2], oracle.FAMILY[etype][0]
    N = nn * ndpn
    b = oracle.blocked(etype, res, nn)
    p = oracle.blocked_perm(etype, nn)
    K = _dense(res, N)
    Kb = _dense(b, N)
    assert np.array_equal(Kb, K[np.ix_(p, p)])
    assert np.array_equal(b["R"], res["R"][p])
    assert b["row_ptr"][-1] == res["row_ptr"][-1]
    for r in range(N):   # ascending columns, pattern rows keep their lengths
        c = b["col_idx"][b["row_ptr"][r]:b["row_ptr"][r + 1]]
        assert np.all(np.diff(c) > 0)
        assert len(c) == res["row_ptr"][p[r] + 1] - res["row_ptr"][p[r]]
    # the leading n_u x n_u block is K restricted to the u dofs (the paper's Kuu)
    u = np.array([a * ndpn + c for a in range(nn) for c in range(dim)])
    nu = nn * dim
    assert np.array_equal(Kb[:nu, :nu], K[np.ix_(u, u)])


# ---------------- mixed-order meshes (SURVEY NEXT f2 x f4) ----------------

def test_mixed_perm_hand_example():
    # one BAR3 element: nodes x = 0 (corner), h/2 (midside), h (corner)
    # interleaved [u0 e0 u1 u2 e2] -> blocked [u0 u1 u2 e0 e2]
    mesh = synth.mixed_mesh(synth.BAR3, (1,), 2.0)
    doff = oracle.mixed_dofs(synth.BAR3, 3, mesh.conn)
    assert list(doff) == [0, 2, 3, 5]
    assert list(oracle.mixed_blocked_perm(doff, 1)) == [0, 2, 3, 1, 4]


@pytest.mark.parametrize("etype,n", [(synth.BAR3, (4,)), (synth.QUAD8, (3, 2))])
def test_mixed_blocked_is_symmetric_permutation(etype, n):
    mesh = synth.mixed_mesh(etype, n, 10.0)
    d, k = synth.mixed_fields(mesh)
    res = oracle.mixed_assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn,
                                d, k)
    dim = synth.MFAM[etype][0]
    p = oracle.mixed_blocked_perm(res["doff"], dim)
    N = p.size
    b = oracle.blocked_from_perm(res, p)
    K, Kb = _dense(res, N), _dense(b, N)
    assert np.array_equal(Kb, K[np.ix_(p, p)])
    assert np.array_equal(b["R"], res["R"][p])
    kind = oracle.dof_kind(res["doff"], dim)
    nu = int((kind < dim).sum())
    u = np.nonzero(kind < dim)[0]
    assert np.array_equal(Kb[:nu, :nu], K[np.ix_(u, u)])
    for r in range(N):
        c = b["col_idx"][b["row_ptr"][r]:b["row_ptr"][r + 1]]
        assert np.all(np.diff(c) > 0)
