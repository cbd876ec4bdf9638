"""Multi-process host logic of the N > 1 path on CPU (gloo, world_size 2).

Each rank builds its row-owned slab (owned node layers + one ghost element layer, global
ids), assembles it with the CPU oracle, keeps its owned rows, and the ranks reduce the sums
of squares of R exactly as lgdm_residual_norms does with NCCL.  Checks: the slabs' owned rows
equal the whole-mesh rows bitwise (ghost recompute is sufficient, global column ids), and the
reduced norms equal the whole-mesh norms.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2301_06503_b200 import slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, etype, n, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.small_config(etype, n)
        ndpn = synth.FAM[etype][2]
        sl = slabs.slab(cfg.n, rank, world)
        mesh = synth.structured_mesh(cfg, elem_layers=sl.elem_layers)
        dofs, kappa = synth.fields(cfg, mesh)
        res = oracle.assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn,
                              dofs, kappa)
        ob, oe = sl.owned_local(mesh.node_gid0)
        r0, r1 = ndpn * ob, ndpn * oe
        R = res["R"][r0:r1]
        lo, hi = res["row_ptr"][r0], res["row_ptr"][r1]
        cols_global = res["col_idx"][lo:hi].astype(np.int64) + ndpn * mesh.node_gid0
        # partial sums of squares (u rows, ebar rows) -> allreduce(sum), as lgdm_residual_norms
        dim = synth.FAM[etype][0]
        comp = np.arange(r0, r1) % ndpn
        part = torch.tensor([np.sum(R[comp != dim] ** 2), np.sum(R[comp == dim] ** 2)],
                            dtype=torch.float64)
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        q.put((rank, sl.owned_nodes, res["row_ptr"][r0:r1 + 1] - lo, cols_global,
               res["val"][lo:hi], R, np.sqrt(part.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("etype,n", [(synth.QUAD4, (9, 11)), (synth.HEX8, (3, 4, 7))])
def test_two_rank_slabs_gloo(etype, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, etype, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.small_config(etype, n)
    ndpn = synth.FAM[etype][2]
    mesh = synth.structured_mesh(cfg)
    dofs, kappa = synth.fields(cfg, mesh)
    full = oracle.assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn,
                           dofs, kappa)
    norms = oracle.residual_norms(etype, full["R"])
    covered = 0
    for rank, (b, e), rp, cols, val, R, rnorm in out:
        r0, r1 = ndpn * b, ndpn * e
        lo, hi = full["row_ptr"][r0], full["row_ptr"][r1]
        np.testing.assert_array_equal(rp, full["row_ptr"][r0:r1 + 1] - lo)
        np.testing.assert_array_equal(cols, full["col_idx"][lo:hi])
        np.testing.assert_array_equal(val, full["val"][lo:hi])
        np.testing.assert_array_equal(R, full["R"][r0:r1])
        np.testing.assert_allclose(rnorm, norms, rtol=1e-13)
        covered += e - b
    assert covered == mesh.coords.shape[0]


def _mixed_worker(rank, world, port, etype, n, q):
    import torch
    from paper_2301_06503_b200 import slabs as sl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        whole = synth.mixed_mesh(etype, n, 10.0)
        dofs_all, kap_all = synth.mixed_fields(whole)
        S = sl.mixed_slab(etype, n, rank, world)
        (nb, ne), (eb, ee), (ob, oe) = S.node_range, S.elem_range, S.owned_local
        conn = whole.conn[eb:ee] - nb
        doff_w = oracle.mixed_dofs(etype, whole.coords.shape[0], whole.conn)
        dofs = dofs_all[doff_w[nb]:doff_w[ne]]
        res = oracle.mixed_assemble(etype, oracle.material(**synth.MATERIAL), whole.coords[nb:ne],
                                    conn, dofs, kap_all[eb:ee])
        d = res["doff"]
        r0, r1 = d[ob], d[oe]
        lo, hi = res["row_ptr"][r0], res["row_ptr"][r1]
        dim = synth.MFAM[etype][0]
        kind = oracle.dof_kind(d, dim)[r0:r1]
        R = res["R"][r0:r1]
        part = torch.tensor([np.sum(R[kind < dim] ** 2), np.sum(R[kind == dim] ** 2)],
                            dtype=torch.float64)
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        q.put((rank, S.global_dof_offset + r0, res["row_ptr"][r0:r1 + 1] - lo,
               res["col_idx"][lo:hi].astype(np.int64) + S.global_dof_offset, res["val"][lo:hi],
               R, np.sqrt(part.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("etype,n", [(synth.QUAD8, (7, 6)), (synth.BAR3, (13,))])
def test_mixed_slabs_gloo(etype, n):
    """mixed-order slabs (slabs.mixed_slab): the owned rows of each rank's local assembly, with
    the global dof offset, equal the whole mesh's rows; reduced norms equal the whole norms"""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mixed_worker, args=(r, world, port, etype, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    whole = synth.mixed_mesh(etype, n, 10.0)
    dofs, kap = synth.mixed_fields(whole)
    ref = oracle.mixed_assemble(etype, oracle.material(**synth.MATERIAL), whole.coords, whole.conn,
                                dofs, kap)
    rp = ref["row_ptr"]
    nxt = 0
    for rank, g0, rpl, cols, val, R, norms in got:
        assert g0 == nxt
        g1 = g0 + R.size
        assert np.array_equal(rpl, rp[g0:g1 + 1] - rp[g0])
        assert np.array_equal(cols, ref["col_idx"][rp[g0]:rp[g1]])
        assert np.array_equal(val, ref["val"][rp[g0]:rp[g1]])
        assert np.array_equal(R, ref["R"][g0:g1])
        nxt = g1
    assert nxt == ref["R"].size
    dim = synth.MFAM[etype][0]
    kind = oracle.dof_kind(ref["doff"], dim)
    want = [np.linalg.norm(ref["R"][kind < dim]), np.linalg.norm(ref["R"][kind == dim])]
    np.testing.assert_allclose(got[0][6], want, rtol=1e-14)


# ---------------- multi-rank Newton pieces: the contract of lgdm_solve ----------------

def _halo_counts(ob, oe, nl, rank, world):
    """The halo counts lgdm_set_comm derives from the all-gathered slab layouts (dofs): my lower
    ghosts come from rank - 1's last owned dofs, my first owned dofs are its upper ghosts (and
    mirrored above); the two directions may differ (mixed-order slabs)."""
    lay = [None] * world
    dist.all_gather_object(lay, (ob, oe, nl))
    send_lo = lay[rank - 1][2] - lay[rank - 1][1] if rank > 0 else 0
    send_hi = lay[rank + 1][0] if rank + 1 < world else 0
    return send_lo, ob, send_hi, nl - oe


def _halo(x, ob, oe, rank, counts):
    """The ghost-dof exchange of lgdm_api.cu halo_exchange with the counts above."""
    import torch
    sl, rl, sh, rh = counts
    reqs, t = [], {}
    if sl > 0:
        t["sl"] = torch.from_numpy(x[ob:ob + sl].copy())
        reqs.append(dist.isend(t["sl"], rank - 1))
    if rl > 0:
        t["rl"] = torch.empty(rl, dtype=torch.float64)
        reqs.append(dist.irecv(t["rl"], rank - 1))
    if sh > 0:
        t["sh"] = torch.from_numpy(x[oe - sh:oe].copy())
        reqs.append(dist.isend(t["sh"], rank + 1))
    if rh > 0:
        t["rh"] = torch.empty(rh, dtype=torch.float64)
        reqs.append(dist.irecv(t["rh"], rank + 1))
    for r in reqs:
        r.wait()
    if rl > 0:
        x[ob - rl:ob] = t["rl"].numpy()
    if rh > 0:
        x[oe:oe + rh] = t["rh"].numpy()


def _solve_slab(rank, world, rp, cols, val, R, ob, oe, nl, col_off, fixed_g, inc_g):
    """lgdm_apply_dirichlet (global ids) + lgdm_solve (Jacobi-BiCGSTAB on the owned rows, local
    vectors with ghosts, halo exchange before each SpMV, allreduced dots) on one rank's rows;
    returns the local delta with its ghosts filled."""
    import torch
    nrow = oe - ob
    counts = _halo_counts(ob, oe, nl, rank, world)
    mask = np.zeros(nl, bool)
    inc = np.zeros(nl)
    loc = fixed_g - col_off
    keep = (loc >= 0) & (loc < nl)
    mask[loc[keep]] = True
    inc[loc[keep]] = inc_g[keep]
    grow = col_off + ob + np.arange(nrow)
    for r in range(nrow):                       # k_dirichlet, row by row
        s = slice(rp[r], rp[r + 1])
        if mask[ob + r]:
            val[s] = np.where(cols[s] == grow[r], 1.0, 0.0)
            R[r] = inc[ob + r]
        else:
            cl = cols[s] - col_off
            f = mask[cl]
            R[r] -= np.dot(val[s][f], inc[cl[f]])
            val[s][f] = 0.0
    diag = np.array([val[rp[r]:rp[r + 1]][cols[rp[r]:rp[r + 1]] == grow[r]][0] for r in range(nrow)])

    def spmv(xl):
        _halo(xl, ob, oe, rank, counts)
        y = np.zeros(nrow)
        for r in range(nrow):
            s = slice(rp[r], rp[r + 1])
            y[r] = np.dot(val[s], xl[cols[s] - col_off])
        return y

    def dot(a, b):
        t = torch.tensor([float(np.dot(a, b))], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    delta, ph, sh = np.zeros(nl), np.zeros(nl), np.zeros(nl)
    r_, r0 = R.copy(), R.copy()
    p_, v = np.zeros(nrow), np.zeros(nrow)
    rho = alpha = omega = 1.0
    bnorm = np.sqrt(dot(R, R))
    for _ in range(4000):
        rho_new = dot(r0, r_)
        beta = (rho_new / rho) * (alpha / omega)
        p_ = r_ + beta * (p_ - omega * v)
        ph[ob:oe] = p_ / diag
        v = spmv(ph)
        alpha = rho_new / dot(r0, v)
        s_ = r_ - alpha * v
        if np.sqrt(dot(s_, s_)) / bnorm <= 1e-12:
            delta[ob:oe] += alpha * ph[ob:oe]
            break
        sh[ob:oe] = s_ / diag
        t_ = spmv(sh)
        omega = dot(t_, s_) / dot(t_, t_)
        delta[ob:oe] += alpha * ph[ob:oe] + omega * sh[ob:oe]
        r_ = s_ - omega * t_
        rho = rho_new
        if np.sqrt(dot(r_, r_)) / bnorm <= 1e-12:
            break
    spmv(delta)                                   # fills the ghost dofs of delta
    return delta


def _newton_worker(rank, world, port, etype, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if etype in (synth.QUAD8, synth.BAR3):    # mixed-order slab (asymmetric ghosts)
            from paper_2301_06503_b200 import slabs as sl
            whole = synth.mixed_mesh(etype, n, 10.0)
            dofs_all, kap_all = synth.mixed_fields(whole)
            dofs_all = 0.0 * dofs_all    # the first Newton iterate (Jacobi-BiCGSTAB stagnates on
            #                              the damaged, loading states of this small mesh)
            S = sl.mixed_slab(etype, n, rank, world)
            (nb, ne), (eb, ee), (obn, oen) = S.node_range, S.elem_range, S.owned_local
            doff_w = oracle.mixed_dofs(etype, whole.coords.shape[0], whole.conn)
            res = oracle.mixed_assemble(etype, oracle.material(**synth.MATERIAL), whole.coords[nb:ne],
                                        whole.conn[eb:ee] - nb, dofs_all[doff_w[nb]:doff_w[ne]],
                                        kap_all[eb:ee])
            d = res["doff"]
            ob, oe, nl, col_off = int(d[obn]), int(d[oen]), int(d[-1]), S.global_dof_offset
            dim = synth.MFAM[etype][0]
            row0 = 2 * n[0] + 1 if etype == synth.QUAD8 else 1          # bottom lattice row / left end
            fixed_g = np.concatenate([doff_w[np.arange(row0)] + c for c in range(dim)])
        else:
            cfg = synth.small_config(etype, n)
            dim, _, ndpn, _ = synth.FAM[etype]
            S = slabs.slab(cfg.n, rank, world)
            mesh = synth.structured_mesh(cfg, elem_layers=S.elem_layers)
            dofs, kappa = synth.fields(cfg, mesh)
            res = oracle.assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn,
                                  dofs, kappa)
            nb, ne_ = S.owned_local(mesh.node_gid0)
            ob, oe, nl = ndpn * nb, ndpn * ne_, ndpn * mesh.coords.shape[0]
            col_off = ndpn * mesh.node_gid0
            layer = int(np.prod([k + 1 for k in cfg.n[:-1]]))    # u dofs of the bottom node layer
            fixed_g = np.concatenate([ndpn * np.arange(layer) + c for c in range(dim)])
        lo, hi = res["row_ptr"][ob], res["row_ptr"][oe]
        rp = res["row_ptr"][ob:oe + 1] - lo
        cols = res["col_idx"][lo:hi].astype(np.int64) + col_off    # global dof ids
        delta = _solve_slab(rank, world, rp, cols, res["val"][lo:hi].copy(), res["R"][ob:oe].copy(),
                            ob, oe, nl, col_off, fixed_g, np.full(fixed_g.size, 1e-3))
        q.put((rank, col_off, ob, oe, delta))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("etype,n", [(synth.QUAD4, (6, 8)), (synth.HEX8, (3, 2, 5)), (synth.QUAD8, (5, 6))])
def test_two_rank_newton_solve_gloo(etype, n):
    """lgdm_solve across 2 ranks (halo exchange of the ghost dofs, allreduced dots, global-id
    Dirichlet) reproduces the one-system solve of the eliminated whole-mesh system, on every
    local dof -- owned and ghost (what lgdm_add_dofs then adds).  QUAD8: mixed-order slabs keep
    two lattice rows of ghosts below and one above, so the two exchange directions differ."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_newton_worker, args=(r, world, port, etype, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if etype == synth.QUAD8:
        whole = synth.mixed_mesh(etype, n, 10.0)
        dofs, kappa = synth.mixed_fields(whole)
        full = oracle.mixed_assemble(etype, oracle.material(**synth.MATERIAL), whole.coords,
                                     whole.conn, 0.0 * dofs, kappa)
        doff_w = oracle.mixed_dofs(etype, whole.coords.shape[0], whole.conn)
        fixed = np.concatenate([doff_w[np.arange(2 * n[0] + 1)] + c for c in range(2)])
        # rank 1 keeps more ghost dofs below than rank 0 keeps above: the directions differ
        assert out[1][2] > out[0][4].size - out[0][3]
    else:
        cfg = synth.small_config(etype, n)
        dim, _, ndpn, _ = synth.FAM[etype]
        mesh = synth.structured_mesh(cfg)
        dofs, kappa = synth.fields(cfg, mesh)
        full = oracle.assemble(etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn, dofs, kappa)
        layer = int(np.prod([k + 1 for k in cfg.n[:-1]]))
        fixed = np.concatenate([ndpn * np.arange(layer) + c for c in range(dim)])
    K = sp.csr_matrix((full["val"], full["col_idx"], full["row_ptr"])).tolil()
    Rf = full["R"].copy()
    inc = np.zeros(Rf.size)
    inc[fixed] = 1e-3
    Rf -= K[:, fixed] @ inc[fixed]
    for d in fixed:
        K[:, d] = 0.0
        K[d, :] = 0.0
        K[d, d] = 1.0
        Rf[d] = 1e-3
    ref = spla.spsolve(K.tocsr(), Rf)
    for rank, col_off, ob, oe, delta in out:
        # BiCGSTAB stops at a 1e-12 relative residual: entries far below the solution scale
        # carry an absolute error of that order times the conditioning (~1e5 for QUAD8)
        np.testing.assert_allclose(delta, ref[col_off:col_off + delta.size], rtol=1e-8,
                                   atol=1e-10 * np.abs(ref).max())