"""CPU oracle for the LGDM K/R assembly path (arXiv 2301.06503) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product
(``paper_2301_06503_b200``) never imports it; the two share no code.

Thin ctypes wrapper over ``liblgdm_oracle.so`` (plain C++, built from
``lgdm_oracle.cpp`` with ``-O2 -ffp-contract=off``).  Every function cites the
PAPER.md passage it implements in the C++ source.  Parity pins live in
``tests/test_oracle_*.py``.

Parity unpinned: physical fidelity to the paper's load-displacement
and damage figures (images and parameters missing from PAPER.md).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lgdm_oracle.cpp")
_HDR = os.path.join(_HERE, "lgdm_oracle.h")
_LIB = os.path.join(_HERE, "liblgdm_oracle.so")

BAR2, QUAD4, HEX8 = 1, 2, 3
# type -> (dim, nen, ndpn, nv, ngp, ndofe)
FAMILY = {1: (1, 2, 2, 1, 2, 4), 2: (2, 4, 3, 3, 4, 12), 3: (3, 8, 4, 6, 8, 32)}


class Material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("k", C.c_double),
                ("kappa0", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("h", C.c_double), ("h_sigma", C.c_double), ("c", C.c_double),
                ("R", C.c_double), ("n", C.c_double), ("t", C.c_double),
                ("eq_variant", C.c_int32), ("pad_", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile the oracle (g++, no FMA contraction, no fast-math)."""
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-fopenmp", "-shared", "-o", _LIB, _SRC]
        subprocess.check_call(cmd, cwd=_HERE)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        i64p = C.POINTER(C.c_int64)
        i32p = C.POINTER(C.c_int32)
        mp = C.POINTER(Material)
        L.oracle_damage.argtypes = [mp, C.c_double, dp, dp]
        L.oracle_interaction.argtypes = [mp, C.c_double, dp, dp]
        L.oracle_eqstrain.argtypes = [mp, C.c_int, dp, dp, dp, dp]
        L.oracle_gauss.argtypes = [C.c_int, dp, dp]
        L.oracle_shape.argtypes = [C.c_int, dp, dp, dp]
        L.oracle_element.argtypes = [C.c_int, mp, dp, dp, dp, dp, dp, dp, dp, i32p]
        L.oracle_pattern_nnz.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p]
        L.oracle_pattern_nnz.restype = C.c_int64
        L.oracle_pattern.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p, i64p, i32p]
        L.oracle_assemble.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p, dp, dp,
                                      i64p, i32p, dp, dp, dp, i64p]
        L.oracle_assemble_d.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p, dp, dp,
                                        dp, dp, i64p, i32p, dp, dp, dp, i64p]
        L.oracle_sdv_width.argtypes = [C.c_int]
        L.oracle_update_state.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p, dp, dp,
                                          dp, dp, dp]
        L.oracle_rows_nnz.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p, C.c_int64, i64p]
        L.oracle_rows_nnz.restype = C.c_int64
        L.oracle_assemble_rows.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p, dp, dp,
                                           C.c_int64, i64p, i64p, i32p, dp, dp, dp]
        L.oracle_update_history.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p, dp, dp]
        L.oracle_residual_norms.argtypes = [C.c_int, C.c_int64, dp, dp]
        L.oracle_mixed_family.argtypes = [C.c_int, i32p]
        L.oracle_mixed_gauss.argtypes = [C.c_int, dp, dp]
        L.oracle_mixed_shape_u.argtypes = [C.c_int, dp, dp, dp]
        L.oracle_mixed_shape_e.argtypes = [C.c_int, dp, dp, dp]
        L.oracle_mixed_element.argtypes = [C.c_int, mp, dp, dp, dp, dp, dp, dp, dp, dp, dp]
        L.oracle_mixed_dofs.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p, i64p]
        L.oracle_mixed_dofs.restype = C.c_int64
        L.oracle_mixed_pattern.argtypes = [C.c_int, C.c_int64, C.c_int64, i64p, i64p, i64p, i32p]
        L.oracle_mixed_pattern.restype = C.c_int64
        L.oracle_mixed_assemble.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p, i64p,
                                            dp, dp, dp, dp, i64p, i32p, dp, dp, dp]
        L.oracle_mixed_update_history.argtypes = [C.c_int, C.c_int64, i64p, i64p, dp, dp]
        L.oracle_mixed_update_state.argtypes = [C.c_int, mp, C.c_int64, dp, C.c_int64, i64p,
                                                i64p, dp, dp, dp, dp, dp]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def material(**kw) -> Material:
    m = Material()
    for k, v in kw.items():
        setattr(m, k, v)
    return m


def damage(m: Material, kappa: float):
    D, dD = C.c_double(), C.c_double()
    lib().oracle_damage(C.byref(m), kappa, C.byref(D), C.byref(dD))
    return D.value, dD.value


def interaction(m: Material, D: float):
    g, dg = C.c_double(), C.c_double()
    lib().oracle_interaction(C.byref(m), D, C.byref(g), C.byref(dg))
    return g.value, dg.value


def eqstrain(m: Material, dim: int, eps_v):
    nv = {1: 1, 2: 3, 3: 6}[dim]
    ev = np.ascontiguousarray(eps_v, dtype=np.float64)
    assert ev.shape == (nv,)
    e = C.c_double()
    d = np.zeros(nv)
    H = np.zeros((nv, nv))
    lib().oracle_eqstrain(C.byref(m), dim, _d(ev), C.byref(e), _d(d), _d(H))
    return e.value, d, H


def gauss(etype: int):
    dim = FAMILY[etype][0]
    xi = np.zeros((8, dim))
    w = np.zeros(8)
    ng = lib().oracle_gauss(etype, _d(xi), _d(w))
    return xi[:ng].copy(), w[:ng].copy()


def shape(etype: int, xi):
    dim, nen = FAMILY[etype][0], FAMILY[etype][1]
    x = np.ascontiguousarray(xi, dtype=np.float64).reshape(dim)
    N = np.zeros(nen)
    dN = np.zeros((nen, dim))
    lib().oracle_shape(etype, _d(x), _d(N), _d(dN))
    return N, dN


def element(etype: int, m: Material, Xe, Ue, kap):
    """Element blocks: returns (Ke [ndofe,ndofe], Fe, Fabs, sigma [ngp,nv], guard [ngp])."""
    dim, nen, ndpn, nv, ngp, nd = FAMILY[etype]
    Xe = np.ascontiguousarray(Xe, dtype=np.float64).reshape(nen, dim)
    Ue = np.ascontiguousarray(Ue, dtype=np.float64).reshape(nen * ndpn)
    kap = np.ascontiguousarray(kap, dtype=np.float64).reshape(ngp)
    Ke = np.zeros((nd, nd))
    Fe = np.zeros(nd)
    Fa = np.zeros(nd)
    sig = np.zeros((ngp, nv))
    guard = np.zeros(ngp, dtype=np.int32)
    rc = lib().oracle_element(etype, C.byref(m), _d(Xe), _d(Ue), _d(kap), _d(Ke), _d(Fe),
                              _d(Fa), _d(sig), _i32(guard))
    if rc != 0:
        raise ValueError(f"oracle_element: det J <= 0 at GP {-rc - 1}")
    return Ke, Fe, Fa, sig, guard


def pattern(etype: int, n_nodes: int, conn):
    ndpn = FAMILY[etype][2]
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    ne = conn.shape[0]
    nnz = lib().oracle_pattern_nnz(etype, n_nodes, ne, _i64(conn))
    rp = np.zeros(n_nodes * ndpn + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int32)
    lib().oracle_pattern(etype, n_nodes, ne, _i64(conn), _i64(rp), _i32(ci))
    return rp, ci


def _opt(a, n):
    """optional per-GP array -> (keep-alive array or None, pointer or None)"""
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise ValueError(f"per-GP array of {a.size} values, expected {n}")
    return a, _d(a)


def assemble(etype: int, m: Material, coords, conn, dofs, kappa, row_ptr=None, col_idx=None,
             kappa0_gp=None, alpha_gp=None):
    """Alg. 1 assembly.  Returns dict(row_ptr, col_idx, val, R, S, n_guard).
    kappa0_gp / alpha_gp: optional per-GP damage threshold and alpha (defect regions)."""
    dim, nen, ndpn, nv, ngp, nd = FAMILY[etype]
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    nn = coords.shape[0]
    ne = conn.shape[0]
    if row_ptr is None:
        row_ptr, col_idx = pattern(etype, nn, conn)
    val = np.zeros(int(row_ptr[-1]))
    R = np.zeros(nn * ndpn)
    S = np.zeros(nn * ndpn)
    ng = C.c_int64()
    k0a, k0p = _opt(kappa0_gp, ne * ngp)
    ala, alp = _opt(alpha_gp, ne * ngp)
    rc = lib().oracle_assemble_d(etype, C.byref(m), nn, _d(coords), ne, _i64(conn), _d(dofs),
                                 _d(kappa), k0p, alp, _i64(row_ptr), _i32(col_idx), _d(val),
                                 _d(R), _d(S), C.byref(ng))
    if rc != 0:
        raise ValueError(f"oracle_assemble failed rc={rc}")
    return dict(row_ptr=row_ptr, col_idx=col_idx, val=val, R=R, S=S, n_guard=ng.value)


def assemble_colored(etype: int, m: Material, coords, conn, dofs, kappa, colour, n_colours,
                     row_ptr=None, col_idx=None, nthreads: int = 0):
    """The Alg. 1 element loop on all host cores, colour by colour (elements of one colour
    share no node).  CPU-baseline timing only; sums in (colour, element) order.  Returns
    dict(row_ptr, col_idx, val, R, S, threads)."""
    dim, nen, ndpn, nv, ngp, nd = FAMILY[etype]
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    colour = np.ascontiguousarray(colour, dtype=np.int32)
    nn, ne = coords.shape[0], conn.shape[0]
    if row_ptr is None:
        row_ptr, col_idx = pattern(etype, nn, conn)
    val = np.zeros(int(row_ptr[-1]))
    R = np.zeros(nn * ndpn)
    S = np.zeros(nn * ndpn)
    th = C.c_int()
    rc = lib().oracle_assemble_colored(etype, C.byref(m), nn, _d(coords), ne, _i64(conn), _d(dofs),
                                       _d(kappa), colour.ctypes.data_as(C.POINTER(C.c_int32)),
                                       int(n_colours), _i64(row_ptr), _i32(col_idx), _d(val), _d(R),
                                       _d(S), int(nthreads), C.byref(th))
    if rc != 0:
        raise ValueError(f"oracle_assemble_colored failed rc={rc}")
    return dict(row_ptr=row_ptr, col_idx=col_idx, val=val, R=R, S=S, threads=th.value)


def assemble_rows(etype: int, m: Material, coords, conn, dofs, kappa, sel_nodes):
    """Block-rows of the selected nodes only (sampled parity at full size)."""
    dim, nen, ndpn, nv, ngp, nd = FAMILY[etype]
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    sel = np.ascontiguousarray(sel_nodes, dtype=np.int64)
    nn, ne, ns = coords.shape[0], conn.shape[0], sel.shape[0]
    nnz = lib().oracle_rows_nnz(etype, nn, ne, _i64(conn), ns, _i64(sel))
    rp = np.zeros(ns * ndpn + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int32)
    val = np.zeros(nnz)
    R = np.zeros(ns * ndpn)
    S = np.zeros(ns * ndpn)
    rc = lib().oracle_assemble_rows(etype, C.byref(m), nn, _d(coords), ne, _i64(conn), _d(dofs),
                                    _d(kappa), ns, _i64(sel), _i64(rp), _i32(ci), _d(val), _d(R),
                                    _d(S))
    if rc != 0:
        raise ValueError(f"oracle_assemble_rows failed rc={rc}")
    return dict(row_ptr=rp, col_idx=ci, val=val, R=R, S=S)


def update_history(etype: int, conn, dofs, kappa):
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    k = np.array(kappa, dtype=np.float64, copy=True)
    ndpn = FAMILY[etype][2]
    lib().oracle_update_history(etype, dofs.size // ndpn, conn.shape[0], _i64(conn), _d(dofs),
                                _d(k))
    return k


def residual_norms(etype: int, R):
    R = np.ascontiguousarray(R, dtype=np.float64)
    out = np.zeros(2)
    lib().oracle_residual_norms(etype, R.size, _d(R), _d(out))
    return out


def sdv_width(etype: int) -> int:
    """doubles per (element, GP) state record: 3 nv + 5"""
    return lib().oracle_sdv_width(etype)


def update_state(etype: int, m: Material, coords, conn, dofs, kappa, kappa0_gp=None,
                 alpha_gp=None):
    """State-variable update (Alg. 2 l.8-14, Fig. 9a).  Returns (sdv [ne, ngp, W], kappa_new);
    record = [eps_v (nv), d eeq/d eps_v (nv), sigma (nv), eeq, ebar, kappa, D, g]."""
    dim, nen, ndpn, nv, ngp, nd = FAMILY[etype]
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    k = np.array(kappa, dtype=np.float64, copy=True).reshape(-1)
    ne = conn.shape[0]
    W = sdv_width(etype)
    sdv = np.zeros(ne * ngp * W)
    k0a, k0p = _opt(kappa0_gp, ne * ngp)
    ala, alp = _opt(alpha_gp, ne * ngp)
    rc = lib().oracle_update_state(etype, C.byref(m), coords.shape[0], _d(coords), ne, _i64(conn),
                                   _d(dofs), _d(k), k0p, alp, _d(sdv))
    if rc != 0:
        raise ValueError(f"oracle_update_state failed rc={rc}")
    return sdv.reshape(ne, ngp, W), k


def blocked_perm(etype: int, n_nodes: int):
    """Blocked DOF order of the paper's global vector [u; ebar] (`u(1:ndof_u)`
    then the ebar dofs): blocked index -> node-interleaved index."""
    dim, ndpn = FAMILY[etype][0], FAMILY[etype][2]
    nu = n_nodes * dim
    r = np.arange(n_nodes * ndpn)
    return np.where(r < nu, (r // dim) * ndpn + r % dim, (r - nu) * ndpn + dim).astype(np.int64)


def blocked(etype: int, res: dict, n_nodes: int):
    """P K P^T and P R of an assembled (node-interleaved) result, columns ascending per row,
    explicit zeros of the pattern kept (reading R-PAT).  Plain definition: a symmetric
    permutation of the CSR, done on the matrix of 1-based source positions (scipy.sparse as
    the primitive) so that every stored entry moves exactly once."""
    return blocked_from_perm(res, blocked_perm(etype, n_nodes))


def blocked_from_perm(res: dict, p):
    """P K P^T and P R for a permutation p (new index -> old index), columns ascending, every
    stored entry moved exactly once (see blocked)."""
    import scipy.sparse as sp
    p = np.asarray(p, dtype=np.int64)
    n = p.size
    nnz = res["val"].size
    pos = sp.csr_matrix((np.arange(1, nnz + 1, dtype=np.float64),
                         res["col_idx"].astype(np.int64), res["row_ptr"]), shape=(n, n))
    Pb = pos[p][:, p].tocsr()
    Pb.sort_indices()
    src = Pb.data.astype(np.int64) - 1
    assert Pb.nnz == nnz and np.array_equal(np.sort(src), np.arange(nnz))
    return dict(row_ptr=Pb.indptr.astype(np.int64), col_idx=Pb.indices.astype(np.int32),
                val=np.asarray(res["val"])[src], R=np.asarray(res["R"])[p])


# ---------------- Newton loop pieces (Alg. 2 l.4-7, l.16) ----------------
# The paper never states its elimination scheme or solver beyond `mldivide`; these are
# the plain definitions of SPEC.md's apply_dirichlet / linear_solve / check_convergence.

def apply_dirichlet(res: dict, fixed, incr):
    """Symmetric elimination of the constrained dofs `fixed` (u dofs) with prescribed increments
    `incr` (the step's displacement increment on the first iteration, 0 afterwards): for every
    free row i, R_i -= sum_j K_ij incr_j over constrained j and K_ij = 0; constrained rows become
    unit rows with R_j = incr_j.  Returns a new dict (row_ptr, col_idx, val, R)."""
    rp, ci = res["row_ptr"], res["col_idx"].astype(np.int64)
    val = np.array(res["val"], dtype=np.float64, copy=True)
    R = np.array(res["R"], dtype=np.float64, copy=True)
    n = R.size
    fixed = np.asarray(fixed, dtype=np.int64)
    inc = np.zeros(n)
    isfix = np.zeros(n, dtype=bool)
    isfix[fixed] = True
    inc[fixed] = np.asarray(incr, dtype=np.float64)
    for i in range(n):
        lo, hi = rp[i], rp[i + 1]
        if isfix[i]:
            val[lo:hi] = np.where(ci[lo:hi] == i, 1.0, 0.0)
            R[i] = inc[i]
        else:
            cols = ci[lo:hi]
            m = isfix[cols]
            R[i] -= float(np.dot(val[lo:hi][m], inc[cols[m]]))
            val[lo:hi][m] = 0.0
    return dict(row_ptr=rp, col_idx=res["col_idx"], val=val, R=R)


def solve(res: dict):
    """Direct sparse solve K delta = R (the paper's mldivide) -- scipy as the primitive."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    n = res["R"].size
    K = sp.csr_matrix((res["val"], res["col_idx"].astype(np.int64), res["row_ptr"]), shape=(n, n))
    return spl.spsolve(K.tocsc(), res["R"])


def converged(etype: int, delta, dofs, tol: float, floor: float = 1e-16):
    """Alg. 1 l.26 / Alg. 2 l.16: ||du|| / max(||u||, floor) <= tol and the same for ebar."""
    dim, ndpn = FAMILY[etype][0], FAMILY[etype][2]
    d = np.asarray(delta).reshape(-1, ndpn)
    u = np.asarray(dofs).reshape(-1, ndpn)
    ru = np.linalg.norm(d[:, :dim]) / max(np.linalg.norm(u[:, :dim]), floor)
    re = np.linalg.norm(d[:, dim]) / max(np.linalg.norm(u[:, dim]), floor)
    return bool(ru <= tol and re <= tol), ru, re


def newton_iteration(etype: int, m: Material, coords, conn, dofs, kappa_hist, fixed, incr):
    """One iteration of Alg. 2 l.4-7: assemble at (dofs, committed history), eliminate the
    constraints, solve, return (delta, dofs + delta)."""
    res = assemble(etype, m, coords, conn, dofs, kappa_hist)
    sys_ = apply_dirichlet(res, fixed, incr)
    delta = solve(sys_)
    return delta, np.asarray(dofs, dtype=np.float64).reshape(-1) + delta


def reaction(res: dict, dof_ids):
    """Reaction at the driven dofs (SPEC reaction_force; the load of the paper's
    load-displacement curves, Fig. 11 / P:418): the internal force sum_i int B^T sigma over the
    listed u dofs of the UNCONSTRAINED assembled system, i.e. -sum R_i (R = F of Eq. 11 has no
    external load in a displacement-controlled problem)."""
    return -float(np.sum(np.asarray(res["R"])[np.asarray(dof_ids, dtype=np.int64)]))


# ---------------------------------------------------------------------------------------
# Mixed-order elements (lgdm_oracle.cpp "Mixed-order elements")
# ---------------------------------------------------------------------------------------
BAR3, QUAD8 = 4, 5


def mixed_family(etype: int):
    """(dim, nenu, nene, nv, ngp, ndofe)"""
    out = np.zeros(6, dtype=np.int32)
    assert lib().oracle_mixed_family(etype, _i32(out)) == 0
    return tuple(int(v) for v in out)


def mixed_gauss(etype: int):
    dim, _, _, _, ngp, _ = mixed_family(etype)
    xi, w = np.zeros(ngp * dim), np.zeros(ngp)
    lib().oracle_mixed_gauss(etype, _d(xi), _d(w))
    return xi.reshape(ngp, dim), w


def mixed_shape(etype: int, xi, field: str = "u"):
    dim, nenu, nene, _, _, _ = mixed_family(etype)
    nen = nenu if field == "u" else nene
    x = np.ascontiguousarray(xi, dtype=np.float64)
    N, dN = np.zeros(nen), np.zeros(nen * dim)
    fn = lib().oracle_mixed_shape_u if field == "u" else lib().oracle_mixed_shape_e
    fn(etype, _d(x), _d(N), _d(dN))
    return N, dN.reshape(nen, dim)


def mixed_element(etype: int, m: Material, Xe, Ue, kap, k0g=None, alg=None):
    dim, nenu, nene, nv, ngp, nd = mixed_family(etype)
    Xe = np.ascontiguousarray(Xe, dtype=np.float64).reshape(-1)
    Ue = np.ascontiguousarray(Ue, dtype=np.float64).reshape(-1)
    kap = np.ascontiguousarray(kap, dtype=np.float64).reshape(-1)
    Ke, Fe, Fa, sig = np.zeros(nd * nd), np.zeros(nd), np.zeros(nd), np.zeros(ngp * nv)
    k0k, k0p = _opt(k0g, ngp)
    alk, alp = _opt(alg, ngp)
    rc = lib().oracle_mixed_element(etype, C.byref(m), _d(Xe), _d(Ue), _d(kap), k0p, alp,
                                    _d(Ke), _d(Fe), _d(Fa), _d(sig))
    if rc != 0:
        raise ValueError(f"oracle_mixed_element rc={rc}")
    return Ke.reshape(nd, nd), Fe, Fa, sig.reshape(ngp, nv)


def mixed_dofs(etype: int, n_nodes: int, conn):
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    doff = np.zeros(n_nodes + 1, dtype=np.int64)
    nd = lib().oracle_mixed_dofs(etype, n_nodes, conn.shape[0], _i64(conn), _i64(doff))
    if nd < 0:
        raise ValueError("inconsistent mixed mesh")
    return doff


def dof_kind(doff, dim: int):
    """component index per global dof: 0..dim-1 displacement, dim = ebar"""
    cnt = np.diff(doff)
    kind = np.concatenate([np.arange(c) for c in cnt]).astype(np.int64)
    return kind


def mixed_pattern(etype: int, n_nodes: int, conn, doff):
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    null = C.POINTER(C.c_int64)()
    nnz = lib().oracle_mixed_pattern(etype, n_nodes, conn.shape[0], _i64(conn), _i64(doff), null,
                                     C.POINTER(C.c_int32)())
    rp = np.zeros(doff[-1] + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int32)
    lib().oracle_mixed_pattern(etype, n_nodes, conn.shape[0], _i64(conn), _i64(doff), _i64(rp),
                               _i32(ci))
    return rp, ci


def mixed_assemble(etype: int, m: Material, coords, conn, dofs, kappa, kappa0_gp=None,
                   alpha_gp=None):
    """Alg. 1 assembly for mixed elements.  Returns dict(row_ptr, col_idx, val, R, S, doff)."""
    dim, nenu, nene, nv, ngp, nd = mixed_family(etype)
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    nn, ne = coords.shape[0], conn.shape[0]
    doff = mixed_dofs(etype, nn, conn)
    rp, ci = mixed_pattern(etype, nn, conn, doff)
    val = np.zeros(ci.size)
    R, S = np.zeros(doff[-1]), np.zeros(doff[-1])
    k0k, k0p = _opt(kappa0_gp, ne * ngp)
    alk, alp = _opt(alpha_gp, ne * ngp)
    rc = lib().oracle_mixed_assemble(etype, C.byref(m), nn, _d(coords), ne, _i64(conn),
                                     _i64(doff), _d(dofs), _d(kappa), k0p, alp, _i64(rp),
                                     _i32(ci), _d(val), _d(R), _d(S))
    if rc != 0:
        raise ValueError(f"oracle_mixed_assemble rc={rc}")
    return dict(row_ptr=rp, col_idx=ci, val=val, R=R, S=S, doff=doff)


def mixed_update_history(etype: int, conn, doff, dofs, kappa):
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    k = np.array(kappa, dtype=np.float64, copy=True)
    lib().oracle_mixed_update_history(etype, conn.shape[0], _i64(conn), _i64(doff), _d(dofs),
                                      _d(k))
    return k


def converged_kind(delta, dofs, kind, dim: int, tol: float, floor: float = 1e-16):
    """Alg. 2 l.16 ratios with the dof kinds of a mixed mesh."""
    d, u = np.asarray(delta), np.asarray(dofs)
    e = kind == dim
    ru = np.linalg.norm(d[~e]) / max(np.linalg.norm(u[~e]), floor)
    re = np.linalg.norm(d[e]) / max(np.linalg.norm(u[e]), floor)
    return bool(ru <= tol and re <= tol), ru, re


def mixed_update_state(etype: int, m: Material, coords, conn, doff, dofs, kappa, kappa0_gp=None,
                       alpha_gp=None):
    """State records [ne, ngp, 3 nv + 5] and the committed kappa (Alg. 2 l.8-14)."""
    dim, nenu, nene, nv, ngp, nd = mixed_family(etype)
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    dofs = np.ascontiguousarray(dofs, dtype=np.float64)
    k = np.array(kappa, dtype=np.float64, copy=True)
    ne = conn.shape[0]
    sdv = np.zeros((ne, ngp, 3 * nv + 5))
    k0k, k0p = _opt(kappa0_gp, ne * ngp)
    alk, alp = _opt(alpha_gp, ne * ngp)
    rc = lib().oracle_mixed_update_state(etype, C.byref(m), coords.shape[0], _d(coords), ne,
                                         _i64(conn), _i64(np.ascontiguousarray(doff)), _d(dofs),
                                         _d(k), k0p, alp, _d(sdv))
    if rc != 0:
        raise ValueError(f"oracle_mixed_update_state rc={rc}")
    return sdv, k


def mixed_blocked_perm(doff, dim: int):
    """Blocked order [u; ebar] of a mixed-order mesh (SPEC DofMap "all displacement
    DOFs, then all micro-strain DOFs"): the u dofs in node order, then the ebar dofs in node
    order.  Returns new index -> node-interleaved index."""
    kind = dof_kind(np.asarray(doff), dim)
    r = np.arange(kind.size)
    return np.concatenate([r[kind < dim], r[kind == dim]])
