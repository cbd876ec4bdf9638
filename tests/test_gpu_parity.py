"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Pattern bit-exact; K within 1e-12 of the row max; R within 1e-12 of S (R-TOL)."""
import numpy as np
import pytest

import oracle
import synth
from paper_2301_06503_b200 import lgdm

from parity import (compare, compare_rows, compare_sampled, gpu_assemble, gpu_rows,
                    oracle_assemble, slice_rows)

pytestmark = pytest.mark.gpu

KERNELS = [lgdm.KERNEL_GENERAL, lgdm.KERNEL_AUTO, lgdm.KERNEL_SWEEP]
SWEEPS = (lgdm.KERNEL_SWEEP,)

CASES = [
    (lgdm.BAR2, (1,)), (lgdm.BAR2, (7,)), (lgdm.BAR2, (100,)),
    (lgdm.QUAD4, (1, 1)), (lgdm.QUAD4, (3, 5)), (lgdm.QUAD4, (37, 29)), (lgdm.QUAD4, (1, 40)),
    (lgdm.QUAD4, (65, 3)),
    (lgdm.HEX8, (1, 1, 1)), (lgdm.HEX8, (3, 4, 5)), (lgdm.HEX8, (17, 9, 11)), (lgdm.HEX8, (1, 1, 9)),
    (lgdm.HEX8, (9, 6, 2)),
]


def _case(etype, n, distort=0.0):
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    coords = synth.distort(mesh, distort) if (distort and etype != lgdm.BAR2) else mesh.coords
    dofs, kappa = synth.fields(cfg, mesh)
    return cfg, mesh, coords, dofs, kappa


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("etype,n", CASES)
def test_parity_small(etype, n, kernel):
    if kernel in SWEEPS and etype == lgdm.BAR2:
        pytest.skip("bar2 has no sweep kernel")
    cfg, mesh, coords, dofs, kappa = _case(etype, n, distort=0.2)
    ref = oracle_assemble(etype, coords, mesh.conn, dofs, kappa)
    assert ref["n_guard"] == 0
    got = gpu_assemble(etype, coords, mesh.conn, dofs, kappa, kernel=kernel)
    compare(ref, got, f"{etype}{n} kernel={kernel}")


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("variant", [dict(h_sigma=0.0), dict(eq_variant=1), dict(h_sigma=7e3, c=0.5, k=3.0, nu=0.3)])
@pytest.mark.parametrize("etype,n", [(lgdm.QUAD4, (11, 8)), (lgdm.HEX8, (5, 4, 3)), (lgdm.BAR2, (9,))])
def test_parity_readings(etype, n, variant, kernel):
    if kernel in SWEEPS and etype == lgdm.BAR2:
        pytest.skip("bar2 has no sweep kernel")
    cfg, mesh, coords, dofs, kappa = _case(etype, n, distort=0.15)
    kw = dict(synth.MATERIAL)
    kw.update(variant)
    ref = oracle_assemble(etype, coords, mesh.conn, dofs, kappa, kw)
    got = gpu_assemble(etype, coords, mesh.conn, dofs, kappa, kw, kernel=kernel)
    compare(ref, got, f"{etype}{n} {variant}")


@pytest.mark.parametrize("kernel", KERNELS)
def test_parity_config0_and_1(kernel):
    for cid in ((1,) if kernel in SWEEPS else (0, 1)):
        cfg = synth.CONFIGS[cid]
        mesh = synth.structured_mesh(cfg)
        dofs, kappa = synth.fields(cfg, mesh)
        ref = oracle_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa)
        got = gpu_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa, kernel=kernel)
        kerr, rerr = compare(ref, got, f"config {cid}")
        print(f"config {cid} kernel {kernel}: max K err/rowmax {kerr:.2e}, max R err/S {rerr:.2e}")


def test_parity_damage_edge_states():
    """All-unloading (kappa_hist = big), all at kappa0 (D = 0), zero field (sqrt guard)."""
    for etype, n in ((lgdm.QUAD4, (6, 5)), (lgdm.HEX8, (3, 3, 2))):
        cfg, mesh, coords, dofs, kappa = _case(etype, n, distort=0.1)
        for dd, kk in ((dofs, np.full_like(kappa, 5e-3)),
                       (dofs * 0.0, np.full_like(kappa, 1e-4)),
                       (dofs * 1e-3, np.full_like(kappa, 1e-4))):
            ref = oracle_assemble(etype, coords, mesh.conn, dd, kk)
            for kernel in KERNELS:
                got = gpu_assemble(etype, coords, mesh.conn, dd, kk, kernel=kernel)
                compare(ref, got, "edge state")


def test_parity_config2_full():
    """BASELINE config 2 (Q4 1000^2, 1 M elements, 81 M entries) in full, default kernel"""
    cfg = synth.CONFIGS[2]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    ref = oracle_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa)
    got = gpu_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa)
    kerr, rerr = compare(ref, got, "config 2 full")
    print(f"config 2 full: max K err/rowmax {kerr:.2e}, max R err/S {rerr:.2e}")


def test_parity_config3_full():
    """BASELINE config 3 (Hex8 100^3, 1 M elements, 436 M entries) in full, default kernel
    (the bench's launch configuration), against the plain serial oracle."""
    cfg = synth.CONFIGS[3]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    ref = oracle_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa)
    got = gpu_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa)
    kerr, rerr = compare(ref, got, "config 3 full")
    print(f"config 3 full: max K err/rowmax {kerr:.2e}, max R err/S {rerr:.2e}")


def config4_sample(cfg, n_nodes, count=10000):
    """Sampled node block-rows of config 4 (Hex8 200^3): random nodes plus forced ones -- the
    first / last node layers, every node layer of a few columns (so every z-chunk boundary of
    the launch), the x / y tile boundaries of the sweep (TX = 3, TY = 7), the mesh corners, and
    nodes whose rows start beyond 2^31 entries."""
    nxN, nyN, nzN = cfg.n[0] + 1, cfg.n[1] + 1, cfg.n[2] + 1
    nid = lambda x, y, z: x + nxN * (y + nyN * z)
    sel = [synth.sample_nodes(n_nodes, count, seed=4)]
    for (x, y) in ((0, 0), (2, 6), (3, 7), (nxN - 1, nyN - 1), (nxN // 2, nyN // 2), (101, 13)):
        sel.append(np.array([nid(x, y, z) for z in range(nzN)]))
    rng = np.random.default_rng(4)
    for z in (0, 1, nzN - 2, nzN - 1):
        xs, ys = rng.integers(0, nxN, 40), rng.integers(0, nyN, 40)
        sel.append(nid(xs, ys, z))
    for xb in (2, 3, 5, 6, 98, 99):          # tile boundaries in x, random y / z
        ys, zs = rng.integers(0, nyN, 30), rng.integers(0, nzN, 30)
        sel.append(nid(xb, ys, zs))
    for yb in (6, 7, 13, 14, 97, 98):        # tile boundaries in y
        xs, zs = rng.integers(0, nxN, 30), rng.integers(0, nzN, 30)
        sel.append(nid(xs, yb, zs))
    sel.append(rng.integers(int(0.7 * n_nodes), n_nodes, 500))   # rows beyond 2^31 entries
    return np.unique(np.concatenate(sel).astype(np.int64))


def test_parity_config4_sampled():
    """The headline workload: BASELINE config 4 (Hex8 200^3, 8 M elements, 3.47 G entries,
    int64 CSR offsets beyond 2^31) at full size in the bench's launch configuration; >= 10^4
    sampled node block-rows (config4_sample) against oracle.assemble_rows, pattern bit-exact,
    K within 1e-12 of the row max, R within 1e-12 of S; total nnz by the closed form."""
    import torch
    cfg = synth.CONFIGS[4]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    n_nodes = mesh.coords.shape[0]
    m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    out = m.assemble()
    torch.cuda.synchronize()
    ndpn = 4
    assert out["nnz"] == ndpn * ndpn * int(np.prod([3 * k + 1 for k in cfg.n])) > 2 ** 31
    sel = config4_sample(cfg, n_nodes)
    assert sel.size >= 10000
    got = gpu_rows(out, sel, ndpn)
    assert (got["row_start"] >= 2 ** 31).sum() > 1000        # int64 offsets exercised
    ref = oracle.assemble_rows(cfg.etype, oracle.material(**synth.MATERIAL), mesh.coords,
                               mesh.conn, dofs, kappa, sel)
    kerr, rerr = compare_rows(ref, got, "config 4 sampled")
    print(f"config 4: {sel.size} sampled nodes, max K err/rowmax {kerr:.2e}, R err/S {rerr:.2e}")
    m.close()


@pytest.mark.parametrize("kernel", [lgdm.KERNEL_SWEEP])
@pytest.mark.parametrize("cid", [2, 3])
def test_parity_full_size_sampled(cid, kernel):
    """BASELINE configs 2 and 3 at full size, in the bench's launch configuration; sampled
    node block-rows against the oracle, pattern checked by the closed-form nnz."""
    cfg = synth.CONFIGS[cid]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    got = gpu_assemble(cfg.etype, mesh.coords, mesh.conn, dofs, kappa, kernel=kernel)
    ndpn = lgdm.FAMILY[cfg.etype][2]
    assert got["row_ptr"][-1] == ndpn * ndpn * int(np.prod([3 * k + 1 for k in cfg.n]))
    sel = synth.sample_nodes(mesh.coords.shape[0], 1500, seed=cid)
    sel = np.unique(np.concatenate([sel, [0, mesh.coords.shape[0] - 1]]))
    ref = oracle.assemble_rows(cfg.etype, oracle.material(**synth.MATERIAL), mesh.coords,
                               mesh.conn, dofs, kappa, sel)
    wk, wr = compare_sampled(ref, got, sel, ndpn)
    print(f"config {cid}: sampled {sel.size} nodes, max K err {wk:.2e}, R err {wr:.2e}")


@pytest.mark.parametrize("kernel", [lgdm.KERNEL_SWEEP])
@pytest.mark.parametrize("etype,n,P", [(lgdm.QUAD4, (23, 31), 3), (lgdm.HEX8, (7, 5, 13), 4),
                                       (lgdm.BAR2, (50,), 2)])
def test_slabs_stitch_bitwise(etype, n, P, kernel):
    """Row-owned slabs with ghost-element recompute: stitched CSR == one-mesh CSR, bitwise."""
    from paper_2301_06503_b200 import slabs
    if kernel in SWEEPS and etype == lgdm.BAR2:
        pytest.skip("bar2 has no sweep kernel")
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    whole = gpu_assemble(etype, mesh.coords, mesh.conn, dofs, kappa, kernel=kernel)
    rows_rp = whole["row_ptr"]
    ndpn = lgdm.FAMILY[etype][2]
    for p in range(P):
        part = slabs.slab(cfg.n, p, P)
        sm = synth.structured_mesh(cfg, elem_layers=part.elem_layers)
        sd, sk = synth.fields(cfg, sm)
        got = gpu_assemble(etype, sm.coords, sm.conn, sd, sk, offset=sm.node_gid0,
                           n_global=cfg.n_nodes, owned=part.owned_local(sm.node_gid0), kernel=kernel)
        r0 = ndpn * part.owned_nodes[0]
        r1 = ndpn * part.owned_nodes[1]
        assert got["first_row"] == r0
        lo, hi = rows_rp[r0], rows_rp[r1]
        np.testing.assert_array_equal(got["row_ptr"], rows_rp[r0:r1 + 1] - lo)
        np.testing.assert_array_equal(got["col_idx"], whole["col_idx"][lo:hi])
        np.testing.assert_array_equal(got["val"], whole["val"][lo:hi])
        np.testing.assert_array_equal(got["R"], whole["R"][r0:r1])


def test_update_history_parity():
    for etype, n in ((lgdm.QUAD4, (30, 20)), (lgdm.HEX8, (6, 5, 4)), (lgdm.BAR2, (40,))):
        cfg, mesh, coords, dofs, kappa = _case(etype, n)
        kappa = np.where(np.arange(kappa.size).reshape(kappa.shape) % 3 == 0, 2e-3, kappa)
        m = lgdm.Mesh(etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
        m.set_state(dofs, kappa)
        m.update_history()
        got = m.get_kappa()
        ref = oracle.update_history(etype, mesh.conn, dofs, kappa)
        unloading = ref == kappa
        np.testing.assert_array_equal(got[unloading], kappa[unloading])
        np.testing.assert_allclose(got[~unloading], ref[~unloading], rtol=1e-14, atol=0)
        assert 0 < (~unloading).sum() < kappa.size
        m.update_history()          # idempotent
        np.testing.assert_array_equal(m.get_kappa(), got)


def test_residual_norms():
    cfg, mesh, coords, dofs, kappa = _case(lgdm.QUAD4, (25, 19))
    ref = oracle_assemble(lgdm.QUAD4, coords, mesh.conn, dofs, kappa)
    expect = oracle.residual_norms(lgdm.QUAD4, ref["R"])
    m = lgdm.Mesh(lgdm.QUAD4, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    m.assemble()
    np.testing.assert_allclose(m.residual_norms(), expect, rtol=1e-10)
    ss = m.residual_sumsq()
    np.testing.assert_allclose(np.sqrt(ss), expect, rtol=1e-10)


def test_determinism_and_device_state():
    import torch
    cfg, mesh, coords, dofs, kappa = _case(lgdm.HEX8, (6, 7, 5))
    m = lgdm.Mesh(lgdm.HEX8, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    a = m.assemble()
    v1 = a["val"].torch().clone()
    r1 = a["R"].torch().clone()
    m.set_state(torch.as_tensor(dofs, device="cuda"), torch.as_tensor(kappa, device="cuda"))
    a = m.assemble()
    assert torch.equal(a["val"].torch(), v1) and torch.equal(a["R"].torch(), r1)


def test_errors():
    cfg, mesh, coords, dofs, kappa = _case(lgdm.QUAD4, (4, 4))
    mat = lgdm.material(**synth.MATERIAL)
    m = lgdm.Mesh(lgdm.QUAD4, coords, mesh.conn, mat)
    with pytest.raises(lgdm.LGDMError) as ei:
        m.assemble()
    assert ei.value.status == 3
    with pytest.raises(lgdm.LGDMError) as ei:
        m.set_state(dofs[:-1], kappa)
    assert ei.value.status == 3
    bad = coords.copy()
    c = mesh.conn[5]
    bad[c[0]], bad[c[2]] = coords[c[2]].copy(), coords[c[0]].copy()   # fold element 5
    with pytest.raises(lgdm.LGDMError) as ei:
        lgdm.Mesh(lgdm.QUAD4, bad, mesh.conn, mat)
    assert ei.value.status == 2 and "element" in str(ei.value)


@pytest.mark.parametrize("kernel", [lgdm.KERNEL_SWEEP])
@pytest.mark.parametrize("etype,n", [(lgdm.QUAD4, (61, 40)), (lgdm.HEX8, (17, 9, 11))])
def test_sweep_bitwise_reproducible(etype, n, kernel):
    """The warp-specialised sweeps hand data between roles through named barriers only and
    sum every entry in a fixed (element layer, colour) order: repeated assemblies -- several
    hundred CTAs in flight -- must agree bitwise (a missing barrier shows up as a difference)."""
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    runs = [gpu_assemble(etype, coords, mesh.conn, dofs, kappa, kernel=kernel) for _ in range(3)]
    for r in runs[1:]:
        np.testing.assert_array_equal(r["val"], runs[0]["val"])
        np.testing.assert_array_equal(r["R"], runs[0]["R"])
