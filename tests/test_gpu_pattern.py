"""A0 on the GPU (lgdm_pattern.cuh) on irregular connectivity, and the lgdm_step graph path.

The structured-grid tests exercise nodes of degree 3 / 9 / 27; here a 'fan' mesh gives a node
shared by 5 quads (11 neighbours) and, extruded, by 10 bricks (33 neighbours) -- more than a
structured grid ever has -- which the general path must assemble exactly like the oracle."""
import numpy as np
import pytest

import oracle
import synth
from paper_2301_06503_b200 import lgdm

from parity import compare, gpu_assemble, oracle_assemble

pytestmark = pytest.mark.gpu


def fan_q4(k=5, r1=1.0, r2=2.2, jitter=0.05, seed=1):
    """k quads around a centre node (valence k): centre 0, spokes 1..k, corners k+1..2k."""
    rng = np.random.default_rng(seed)
    pts = [(0.0, 0.0)]
    for i in range(k):
        a = 2 * np.pi * i / k
        pts.append((r1 * np.cos(a), r1 * np.sin(a)))
    for i in range(k):
        a = 2 * np.pi * (i + 0.5) / k
        pts.append((r2 * np.cos(a), r2 * np.sin(a)))
    X = np.array(pts) + jitter * rng.standard_normal((2 * k + 1, 2))
    X[0] = 0.0
    conn = [(0, 1 + i, 1 + k + i, 1 + (i + 1) % k) for i in range(k)]   # counter-clockwise
    return X, np.array(conn, dtype=np.int64)


def fan_hex8(k=5, layers=2, dz=0.8):
    X2, c2 = fan_q4(k)
    n2 = X2.shape[0]
    X = np.concatenate([np.column_stack([X2, np.full(n2, l * dz)]) for l in range(layers + 1)])
    conn = [np.concatenate([c + l * n2, c + (l + 1) * n2]) for l in range(layers) for c in c2]
    return X, np.array(conn, dtype=np.int64)


def fields(n_nodes, ndpn, n_elems, ngp, seed):
    rng = np.random.default_rng(seed)
    d = 1e-3 * rng.standard_normal((n_nodes, ndpn))
    d[:, -1] = 2e-4 * (1 + 0.3 * rng.random(n_nodes))
    kappa = np.maximum(1e-4, 4e-4 * rng.random((n_elems, ngp)))
    return d, kappa


@pytest.mark.parametrize("etype", [lgdm.QUAD4, lgdm.HEX8])
def test_irregular_fan_general_path(etype):
    X, conn = fan_q4() if etype == lgdm.QUAD4 else fan_hex8()
    dim, nen, ndpn, ngp = lgdm.FAMILY[etype]
    dofs, kappa = fields(X.shape[0], ndpn, conn.shape[0], ngp, seed=etype)
    ref = oracle_assemble(etype, X, conn, dofs, kappa)
    got = gpu_assemble(etype, X, conn, dofs, kappa, kernel=lgdm.KERNEL_AUTO)
    assert got["info"]["structured"] == 0
    # the centre node's degree: 11 (Q4, valence 5) / 33 (Hex8: the middle-layer centre, 10 bricks)
    rp = got["row_ptr"]
    c = 0 if etype == lgdm.QUAD4 else 11
    assert (rp[ndpn * c + 1] - rp[ndpn * c]) // ndpn == (11 if etype == lgdm.QUAD4 else 33)
    compare(ref, got, f"fan {etype}")


def test_pattern_matches_oracle_slab_offsets():
    """Device-built pattern of a row-owned slab (global column ids, owned node range)."""
    from paper_2301_06503_b200 import slabs
    cfg = synth.small_config(lgdm.HEX8, (5, 4, 7))
    full = synth.structured_mesh(cfg)
    rp_ref, ci_ref = oracle.pattern(lgdm.HEX8, full.coords.shape[0], full.conn)
    for p in range(3):
        part = slabs.slab(cfg.n, p, 3)
        sm = synth.structured_mesh(cfg, elem_layers=part.elem_layers)
        d, k = synth.fields(cfg, sm)
        got = gpu_assemble(lgdm.HEX8, sm.coords, sm.conn, d, k, offset=sm.node_gid0,
                           n_global=cfg.n_nodes, owned=part.owned_local(sm.node_gid0),
                           kernel=lgdm.KERNEL_GENERAL)
        r0, r1 = 4 * part.owned_nodes[0], 4 * part.owned_nodes[1]
        lo, hi = rp_ref[r0], rp_ref[r1]
        np.testing.assert_array_equal(got["row_ptr"], rp_ref[r0:r1 + 1] - lo)
        np.testing.assert_array_equal(got["col_idx"], ci_ref[lo:hi])


@pytest.mark.parametrize("etype,n", [(lgdm.QUAD4, (13, 9)), (lgdm.HEX8, (5, 4, 6))])
def test_step_graph_equals_eager(etype, n):
    """lgdm_step: the CUDA-graph replay gives the same K, R, norms and history as the eager
    calls (assemble, residual_norms, update_history), bitwise."""
    import torch
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    mat = lgdm.material(**synth.MATERIAL)
    a = lgdm.Mesh(etype, mesh.coords, mesh.conn, mat)
    b = lgdm.Mesh(etype, mesh.coords, mesh.conn, mat)
    a.set_state(dofs, kappa)
    b.set_state(dofs, kappa)
    for it in range(4):
        a.assemble()
        na = a.residual_norms()
        a.update_history()
        l0 = b.launches
        nb = b.step(graph=True, history=True)
        assert b.launches > l0
        np.testing.assert_array_equal(na, nb)
        np.testing.assert_array_equal(a.get_kappa(), b.get_kappa())
        a.scale_dofs(1.05)
        b.scale_dofs(1.05)
    # K and R of the last graph replay equal an eager assemble of the same state
    ob = b.assemble()
    oa = a.assemble()
    torch.cuda.synchronize()
    assert torch.equal(oa["val"].torch(), ob["val"].torch())
    assert torch.equal(oa["R"].torch(), ob["R"].torch())
    a.close()
    b.close()
