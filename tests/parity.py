"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI, slice the
oracle's CSR, and compare with the tolerances of north_star / DESIGN.md:
  * row_ptr, col_idx bit-exact;
  * K: |dK_ij| <= 1e-12 * max_j |K_ij| (row max of the oracle row);
  * R: |dR_i| <= 1e-12 * S_i, S_i = sum over elements and GPs of |contribution| (reading R-TOL).
"""
import numpy as np

import oracle
import synth
from paper_2301_06503_b200 import lgdm

KTOL = 1e-12
RTOL = 1e-12


def gpu_assemble(etype, coords, conn, dofs, kappa, mat_kw=None, kernel=lgdm.KERNEL_AUTO,
                 offset=0, n_global=None, owned=None):
    import torch
    mat = lgdm.material(**(mat_kw or synth.MATERIAL))
    m = lgdm.Mesh(etype, coords, conn, mat, global_node_offset=offset, n_global_nodes=n_global,
                  owned=owned)
    m.set_kernel(kernel)
    m.set_state(dofs, kappa)
    out = m.assemble()
    torch.cuda.synchronize()
    res = dict(row_ptr=out["row_ptr"].torch().cpu().numpy(),
               col_idx=out["col_idx"].torch().cpu().numpy(),
               val=out["val"].torch().cpu().numpy(), R=out["R"].torch().cpu().numpy(),
               first_row=out["first_row"], info=m.info(), mesh=m)
    return res


def oracle_assemble(etype, coords, conn, dofs, kappa, mat_kw=None):
    return oracle.assemble(etype, oracle.material(**(mat_kw or synth.MATERIAL)), coords, conn,
                           dofs, kappa)


def slice_rows(ref, r0, r1):
    rp = ref["row_ptr"]
    lo, hi = rp[r0], rp[r1]
    return dict(row_ptr=rp[r0:r1 + 1] - lo, col_idx=ref["col_idx"][lo:hi], val=ref["val"][lo:hi],
                R=ref["R"][r0:r1], S=ref["S"][r0:r1])


def compare(ref, got, what=""):
    """Assert parity; returns (max K error / rowmax, max R error / S)."""
    assert np.array_equal(got["row_ptr"], ref["row_ptr"]), f"{what}: row_ptr differs"
    assert np.array_equal(got["col_idx"], ref["col_idx"]), f"{what}: col_idx differs"
    rp = ref["row_ptr"]
    nrows = rp.size - 1
    rows = np.repeat(np.arange(nrows), np.diff(rp))
    absv = np.abs(ref["val"])
    rowmax = np.maximum.reduceat(absv, rp[:-1]) if absv.size else np.zeros(nrows)   # rows are non-empty
    dk = np.abs(got["val"] - ref["val"])
    kerr = dk / np.maximum(rowmax[rows], 1e-300)
    assert np.all(dk <= KTOL * rowmax[rows]), (
        f"{what}: K mismatch, worst {kerr.max():.3e} at entry {kerr.argmax()}")
    dr = np.abs(got["R"] - ref["R"])
    rerr = dr / np.maximum(ref["S"], 1e-300)
    assert np.all(dr <= RTOL * ref["S"] + 1e-300), (
        f"{what}: R mismatch, worst {rerr.max():.3e} at row {rerr.argmax()}")
    return float(kerr.max(initial=0.0)), float(rerr.max(initial=0.0))


def compare_sampled(ref_rows, got, sel_nodes, ndpn, owned_begin=0):
    """Parity on sampled node block-rows: ref_rows from oracle.assemble_rows."""
    rp = got["row_ptr"]
    worst_k = worst_r = 0.0
    for s, a in enumerate(sel_nodes):
        for i in range(ndpn):
            r = ndpn * (a - owned_begin) + i
            lo, hi = rp[r], rp[r + 1]
            plo, phi = ref_rows["row_ptr"][s * ndpn + i], ref_rows["row_ptr"][s * ndpn + i + 1]
            assert np.array_equal(got["col_idx"][lo:hi], ref_rows["col_idx"][plo:phi]), (a, i)
            rv = ref_rows["val"][plo:phi]
            rmax = np.abs(rv).max()
            dk = np.abs(got["val"][lo:hi] - rv)
            assert np.all(dk <= KTOL * rmax), (a, i, (dk / rmax).max())
            worst_k = max(worst_k, float((dk / rmax).max()))
            dr = abs(got["R"][r] - ref_rows["R"][s * ndpn + i])
            S = ref_rows["S"][s * ndpn + i]
            assert dr <= RTOL * S + 1e-300, (a, i, dr / S)
            worst_r = max(worst_r, dr / S)
    return worst_k, worst_r


def gpu_rows(out, sel_nodes, ndpn, owned_begin=0):
    """The block-rows of the selected (owned-local) nodes of an assembled system, gathered on the
    device (K can be far larger than what is worth copying to the host): row_ptr / col_idx / val
    restricted to those rows, R, and the int64 offsets of the rows' first entries."""
    import torch
    rp = out["row_ptr"].torch()
    rows = (torch.as_tensor(np.asarray(sel_nodes) - owned_begin, device=rp.device)[:, None] * ndpn +
            torch.arange(ndpn, device=rp.device)[None, :]).reshape(-1)
    lo, hi = rp[rows], rp[rows + 1]
    cnt = hi - lo
    starts = torch.repeat_interleave(lo, cnt)
    first = torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
    idx = starts + (torch.arange(int(cnt.sum()), device=rp.device) - first)
    sub_rp = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=rp.device)
    sub_rp[1:] = torch.cumsum(cnt, 0)
    return dict(row_ptr=sub_rp.cpu().numpy(), col_idx=out["col_idx"].torch()[idx].cpu().numpy(),
                val=out["val"].torch()[idx].cpu().numpy(), R=out["R"].torch()[rows].cpu().numpy(),
                row_start=lo.cpu().numpy())


def compare_rows(ref_rows, got_rows, what=""):
    """Parity of gathered block-rows (gpu_rows) against oracle.assemble_rows of the same nodes,
    row by row: pattern bit-exact, K within KTOL of the oracle row max, R within RTOL of S."""
    assert np.array_equal(got_rows["row_ptr"], ref_rows["row_ptr"]), f"{what}: row lengths differ"
    assert np.array_equal(got_rows["col_idx"], ref_rows["col_idx"]), f"{what}: col_idx differs"
    return compare(dict(row_ptr=ref_rows["row_ptr"], col_idx=ref_rows["col_idx"],
                        val=ref_rows["val"], R=ref_rows["R"], S=ref_rows["S"]),
                   dict(row_ptr=got_rows["row_ptr"], col_idx=got_rows["col_idx"],
                        val=got_rows["val"], R=got_rows["R"]), what)


def record_groups(W):
    """component groups of a state record [eps_v, d eeq/d eps_v, sigma, eeq, ebar, kappa, D, g]"""
    nv = (W - 5) // 3
    strain = list(range(nv)) + [3 * nv, 3 * nv + 1, 3 * nv + 2]
    return [strain, list(range(nv, 2 * nv)), list(range(2 * nv, 3 * nv)), [3 * nv + 3, 3 * nv + 4]]


def check_records(W, got, ref):
    """state records (lgdm_update_state) against the oracle's: per GP record and component
    group, within 1e-12 of the group's largest magnitude in that record"""
    got = got.reshape(-1, W)
    ref = ref.reshape(-1, W)
    worst, where = 0.0, None
    for grp in record_groups(W):
        scale = np.maximum(np.abs(ref[:, grp]).max(axis=1, keepdims=True), 1e-300)   # per record
        err = np.abs(got[:, grp] - ref[:, grp]) / scale
        if err.max() > worst:
            worst = float(err.max())
            r, c = np.unravel_index(err.argmax(), err.shape)
            where = (int(r), grp[c])
    assert worst <= 1e-12, f"worst {worst:.3e} at (GP record, component) {where}"
    return worst
