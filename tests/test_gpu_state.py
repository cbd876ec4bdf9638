"""GPU parity of the state-variable update (lgdm_update_state; Alg. 2
l.8-14, Fig. 9a) and of the per-GP defect fields (lgdm_set_defects) against the CPU
oracle, through the C ABI.

Tolerances (the per-row rule of the K parity carried to the records): within every GP record,
each component within 1e-12 of the largest magnitude of its group in THAT record -- strains
(eps_v, eeq, ebar, kappa), d eeq / d eps_v, stresses, damage (D, g) -- (the FP64 evaluation
orders differ); the committed history within 1e-13 relative
(a copy of ebar -- interpolated in a different FMA order -- or of kappa_hist; both sides take
the same threshold decision on inputs kept away from it); K / R of the defect-field assembly
as in parity.py.
"""
import numpy as np
import pytest

import oracle
import synth
from paper_2301_06503_b200 import lgdm

from parity import check_records, compare

pytestmark = pytest.mark.gpu

CASES = [(lgdm.BAR2, (7,)), (lgdm.QUAD4, (5, 4)), (lgdm.QUAD4, (37, 29)),
         (lgdm.HEX8, (3, 4, 5)), (lgdm.HEX8, (9, 6, 2))]


def _case(etype, n, distort=0.1):
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    coords = synth.distort(mesh, distort) if etype != lgdm.BAR2 else mesh.coords
    dofs, kappa = synth.fields(cfg, mesh)
    return cfg, mesh, coords, dofs, kappa


def _defects(kappa, seed):
    rng = np.random.default_rng(seed)
    k = kappa.reshape(-1)
    # thresholds well away from the state's kappa (both damaging and undamaged GPs)
    k0 = np.where(rng.uniform(size=k.shape) < 0.7, k * rng.uniform(0.3, 0.8, k.shape), k * 1.7)
    al = rng.uniform(0.3, 1.0, k.shape)
    return k0, al


@pytest.mark.parametrize("etype,n", CASES)
@pytest.mark.parametrize("defects", [False, True])
def test_update_state_parity(etype, n, defects):
    import torch
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    k0, al = _defects(kappa, 3 + etype) if defects else (None, None)
    ref, kref = oracle.update_state(etype, oracle.material(**synth.MATERIAL), coords, mesh.conn,
                                    dofs, kappa, kappa0_gp=k0, alpha_gp=al)
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    if defects:
        m.set_defects(k0, al)
    got = m.update_state()
    torch.cuda.synchronize()
    check_records(oracle.sdv_width(etype), got.cpu().numpy(), ref)
    np.testing.assert_allclose(m.get_kappa().reshape(-1), kref.reshape(-1), rtol=1e-13, atol=0)
    # the record's kappa is the committed history
    W = oracle.sdv_width(etype)
    nv = oracle.FAMILY[etype][3]
    assert np.array_equal(got.cpu().numpy().reshape(-1, W)[:, 3 * nv + 2],
                          m.get_kappa().reshape(-1))
    m.close()


def test_update_state_host_destination_and_history_only():
    import torch
    etype, n = lgdm.QUAD4, (6, 5)
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    dev = m.update_state().cpu().numpy()
    m.set_state(dofs, kappa)
    host = np.zeros_like(dev)
    m.update_state(out=host)
    assert np.array_equal(dev, host)
    # NULL destination: history commit only, equal to lgdm_update_history
    m.set_state(dofs, kappa)
    lgdm._check(lgdm.load().lgdm_update_state(m._h, None, 0, 1))
    k1 = m.get_kappa()
    m.set_state(dofs, kappa)
    m.update_history()
    assert np.array_equal(k1, m.get_kappa())
    m.close()


def test_update_state_errors():
    etype, n = lgdm.HEX8, (2, 2, 2)
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    with pytest.raises(lgdm.LGDMError):
        m.update_state()                       # before set_state
    m.set_state(dofs, kappa)
    L = lgdm.load()
    buf = np.zeros(10)
    assert L.lgdm_update_state(m._h, buf.ctypes.data, 10, 0) != 0   # wrong size
    assert L.lgdm_set_defects(m._h, buf.ctypes.data, None, 10, 0) != 0
    assert [lgdm.sdv_width(t) for t in (1, 2, 3)] == [8, 14, 23] and lgdm.sdv_width(9) == -1
    m.close()


@pytest.mark.parametrize("etype,n", [(lgdm.QUAD4, (11, 7)), (lgdm.HEX8, (5, 4, 3))])
def test_defect_assembly_parity(etype, n):
    import torch
    cfg, mesh, coords, dofs, kappa = _case(etype, n)
    k0, al = _defects(kappa, 11 + etype)
    ref = oracle.assemble(etype, oracle.material(**synth.MATERIAL), coords, mesh.conn, dofs,
                          kappa, kappa0_gp=k0, alpha_gp=al)
    plain = oracle.assemble(etype, oracle.material(**synth.MATERIAL), coords, mesh.conn, dofs,
                            kappa)
    assert not np.allclose(ref["val"], plain["val"])
    for kernel in (lgdm.KERNEL_AUTO, lgdm.KERNEL_GENERAL, lgdm.KERNEL_SWEEP):
        m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
        m.set_kernel(kernel)
        m.set_state(dofs, kappa)
        m.set_defects(k0, al)
        out = m.assemble()
        torch.cuda.synchronize()
        got = dict(row_ptr=out["row_ptr"].torch().cpu().numpy(),
                   col_idx=out["col_idx"].torch().cpu().numpy(),
                   val=out["val"].torch().cpu().numpy(), R=out["R"].torch().cpu().numpy())
        compare(ref, got, f"defects kernel {kernel}")
        # clearing the fields returns to the uniform material (and to the sweep path)
        m.set_defects(None, None)
        out = m.assemble()
        torch.cuda.synchronize()
        got = dict(row_ptr=out["row_ptr"].torch().cpu().numpy(),
                   col_idx=out["col_idx"].torch().cpu().numpy(),
                   val=out["val"].torch().cpu().numpy(), R=out["R"].torch().cpu().numpy())
        compare(plain, got, f"cleared kernel {kernel}")
        m.close()


# ---------------- blocked DOF order [u; ebar] ----------------

@pytest.mark.parametrize("etype,n,kernel", [(lgdm.BAR2, (9,), lgdm.KERNEL_AUTO),
                                            (lgdm.QUAD4, (7, 5), lgdm.KERNEL_AUTO),
                                            (lgdm.QUAD4, (7, 5), lgdm.KERNEL_GENERAL),
                                            (lgdm.HEX8, (4, 3, 5), lgdm.KERNEL_AUTO),
                                            (lgdm.HEX8, (3, 2, 2), lgdm.KERNEL_GENERAL)])
def test_blocked_order(etype, n, kernel):
    import torch
    cfg, mesh, coords, dofs, kappa = _case(etype, n, distort=0.0)
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_kernel(kernel)
    m.set_state(dofs, kappa)
    out = m.assemble()
    b = m.get_blocked()
    torch.cuda.synchronize()
    got = {k: out[k].torch().cpu().numpy() for k in ("row_ptr", "col_idx", "val", "R")}
    gb = {k: b[k].torch().cpu().numpy() for k in ("row_ptr", "col_idx", "val", "R")}
    nn = coords.shape[0]
    # a pure permutation of the interleaved result: bit-identical to the oracle's permutation
    # of the same CSR
    ob = oracle.blocked(etype, got, nn)
    for k in ("row_ptr", "col_idx", "val", "R"):
        assert np.array_equal(gb[k], ob[k]), k
    # and within parity of the oracle's own assembly, permuted
    ref = oracle.assemble(etype, oracle.material(**synth.MATERIAL), coords, mesh.conn, dofs, kappa)
    rb = oracle.blocked(etype, ref, nn)
    rb["S"] = ref["S"][oracle.blocked_perm(etype, nn)]
    compare(rb, gb, "blocked")
    m.close()


def test_blocked_errors():
    etype, n = lgdm.QUAD4, (3, 3)
    cfg, mesh, coords, dofs, kappa = _case(etype, n, distort=0.0)
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    with pytest.raises(lgdm.LGDMError):
        m.get_blocked()                       # before assemble
    m.close()
    nn = coords.shape[0]
    m = lgdm.Mesh(etype, coords, mesh.conn, lgdm.material(**synth.MATERIAL),
                  global_node_offset=0, n_global_nodes=nn, owned=(0, nn - 4))
    m.set_state(dofs, kappa)
    m.assemble()
    with pytest.raises(lgdm.LGDMError):
        m.get_blocked()                       # not a whole single-rank mesh
    m.close()


@pytest.mark.parametrize("etype,n", [(lgdm.QUAD4, (12, 9)), (lgdm.HEX8, (5, 4, 6))])
def test_prefetch_dofs_matches_set_state(etype, n):
    """lgdm_prefetch_dofs + lgdm_set_state_prefetched (overlapped input transfer): a sequence of
    iterates gives bit-identical K and R to plain set_state, and misuse is refused"""
    import torch
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    seq = [dofs * s for s in (1.0, 1.3, 0.7)]
    mat = lgdm.material(**synth.MATERIAL)
    ref = lgdm.Mesh(etype, mesh.coords, mesh.conn, mat)
    want = []
    for d in seq:
        ref.set_state(d, kappa)
        out = ref.assemble()
        torch.cuda.synchronize()
        want.append((out["val"].torch().cpu().numpy().copy(), out["R"].torch().cpu().numpy().copy()))
    m = lgdm.Mesh(etype, mesh.coords, mesh.conn, mat)
    with pytest.raises(lgdm.LGDMError):
        m.set_state_prefetched()                      # nothing pending
    m.set_state(seq[0], kappa)
    host = [torch.from_numpy(d.reshape(-1).copy()).pin_memory() for d in seq]
    m.prefetch_dofs(host[0])
    with pytest.raises(lgdm.LGDMError):
        m.prefetch_dofs(host[0])                      # one pending at a time
    for t in range(len(seq)):
        m.set_state_prefetched()
        if t + 1 < len(seq):
            m.prefetch_dofs(host[t + 1])
        out = m.assemble()
        torch.cuda.synchronize()
        assert np.array_equal(out["val"].torch().cpu().numpy(), want[t][0])
        assert np.array_equal(out["R"].torch().cpu().numpy(), want[t][1])
    m.close()
    ref.close()


def test_nccl_single_rank_comm():
    """lgdm_nccl_unique_id + lgdm_set_comm (NCCL dlopen'ed) with one rank: the allreduce of
    lgdm_residual_norms is the identity, so the norms equal the communicator-free ones"""
    cfg = synth.small_config(lgdm.HEX8, (3, 3, 4))
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    mat = lgdm.material(**synth.MATERIAL)
    a = lgdm.Mesh(lgdm.HEX8, mesh.coords, mesh.conn, mat)
    a.set_state(dofs, kappa)
    a.assemble()
    want = a.residual_norms()
    b = lgdm.Mesh(lgdm.HEX8, mesh.coords, mesh.conn, mat)
    b.set_comm(lgdm.nccl_unique_id(), 1, 0)
    b.set_state(dofs, kappa)
    b.assemble()
    got = b.residual_norms()
    assert np.array_equal(got, want)
    a.close()
    b.close()


def test_mesh_on_every_visible_device():
    """One process drives a mesh on every visible GPU (the sweeps' dynamic shared-memory
    attribute is a per-device setting, set once per device) and assembles with the default
    sweep on each; every device gives the same bits."""
    import torch
    etype, n = lgdm.HEX8, (7, 5, 4)
    cfg = synth.small_config(etype, n)
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    outs = []
    for dev in range(torch.cuda.device_count()):
        with torch.cuda.device(dev):
            m = lgdm.Mesh(etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL), device=dev,
                          stream=torch.cuda.current_stream(dev).cuda_stream)
            m.set_kernel(lgdm.KERNEL_SWEEP)
            m.set_state(dofs, kappa)
            o = m.assemble()
            torch.cuda.synchronize(dev)
            outs.append(o["val"].torch(device=f"cuda:{dev}").cpu().numpy())
            m.close()
    assert len(outs) >= 1
    for v in outs[1:]:
        np.testing.assert_array_equal(v, outs[0])


def _state_sample(cfg, n_elems, rng):
    """elements of the bench-size state check: random ones plus the first / last element
    layers and the x / y boundary columns"""
    nx = cfg.n[0]
    per = int(np.prod(cfg.n[:-1]))
    sel = [rng.integers(0, n_elems, 20000), np.arange(min(per, 2000)),
           np.arange(max(n_elems - per, 0), n_elems)[:2000],
           np.arange(0, n_elems, nx)[:3000], np.arange(nx - 1, n_elems, nx)[:3000]]
    return np.unique(np.concatenate(sel).astype(np.int64))


@pytest.mark.parametrize("cid", [2, 4])
def test_update_state_bench_size_sampled(cid):
    """lgdm_update_state at the bench's sizes (BASELINE config 2: Q4 1000^2; config 4: Hex8
    200^3, 64 M GP records) through the same call the bench times; ~3e4 sampled elements'
    records (random + boundary layers / columns) against the oracle, per-record groups as
    above, and the committed history of the sampled GPs."""
    import torch
    cfg = synth.CONFIGS[cid]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    ngp = kappa.reshape(mesh.conn.shape[0], -1).shape[1]
    m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(dofs, kappa)
    got = m.update_state()
    torch.cuda.synchronize()
    sel = _state_sample(cfg, mesh.conn.shape[0], np.random.default_rng(11 + cid))
    got_s = got[torch.as_tensor(sel, device=got.device)].cpu().numpy()
    kap_s = m.get_kappa().reshape(-1, ngp)[sel]
    m.close()
    ref, kref = oracle.update_state(cfg.etype, oracle.material(**synth.MATERIAL), mesh.coords,
                                    mesh.conn[sel], dofs, kappa.reshape(-1, ngp)[sel])
    worst = check_records(oracle.sdv_width(cfg.etype), got_s, ref)
    np.testing.assert_allclose(kap_s.reshape(-1), kref.reshape(-1), rtol=1e-13, atol=0)
    print(f"config {cid}: {sel.size} sampled elements, worst record error / group max {worst:.2e}")
