"""Thin ctypes binding of liblgdm.so (include/lgdm.h) -- argument marshalling only.

Every step of the assembly path runs in the library's CUDA kernels.  There is no CPU
path: if the compiled library is missing, :func:`load` raises.  PyTorch is used only for
device memory views (``__cuda_array_interface__``), streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LGDM_LIB") or os.path.join(_HERE, "liblgdm.so")   # override: experiments

BAR2, QUAD4, HEX8 = 1, 2, 3
BAR3, QUAD8 = 4, 5          # mixed order: quadratic u, linear ebar
# type -> (dim, nen, ndpn, ngp); mixed families: nen = u nodes, ndpn = dofs of a corner node
FAMILY = {BAR2: (1, 2, 2, 2), QUAD4: (2, 4, 3, 4), HEX8: (3, 8, 4, 8),
          BAR3: (1, 3, 2, 3), QUAD8: (2, 8, 3, 9)}
KERNEL_AUTO, KERNEL_GENERAL, KERNEL_SWEEP = 0, 1, 2

STATUS = {0: "LGDM_OK", 1: "LGDM_ERR_INVALID_ARGUMENT", 2: "LGDM_ERR_INVERTED_ELEMENT",
          3: "LGDM_ERR_INVALID_STATE", 4: "LGDM_ERR_OUT_OF_MEMORY", 5: "LGDM_ERR_CUDA",
          6: "LGDM_ERR_NCCL", 7: "LGDM_ERR_UNSUPPORTED", 8: "LGDM_ERR_NOT_CONVERGED"}

# every symbol include/lgdm.h declares
EXPORTS = ["lgdm_create_mesh", "lgdm_set_state", "lgdm_assemble", "lgdm_update_history",
           "lgdm_residual_sumsq", "lgdm_residual_norms", "lgdm_set_comm", "lgdm_nccl_unique_id",
           "lgdm_get_kappa",
           "lgdm_scale_dofs", "lgdm_set_kernel", "lgdm_get_info", "lgdm_launch_count",
           "lgdm_last_error", "lgdm_destroy", "lgdm_sdv_width", "lgdm_set_defects",
           "lgdm_update_state", "lgdm_get_blocked", "lgdm_apply_dirichlet", "lgdm_solve",
           "lgdm_add_dofs", "lgdm_delta_norms", "lgdm_delta_ratios", "lgdm_step", "lgdm_reaction", "lgdm_solve_direct",
           "lgdm_dof_offsets", "lgdm_prefetch_dofs", "lgdm_set_state_prefetched",
           "lgdm_create_mesh_mixed"]


class LGDMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("k", C.c_double),
                ("kappa0", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("h", C.c_double), ("h_sigma", C.c_double), ("c", C.c_double),
                ("R", C.c_double), ("n", C.c_double), ("thickness_or_area", C.c_double),
                ("eq_variant", C.c_int32), ("reserved", C.c_int32)]


class CSR(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("first_row", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("val", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [("elem_type", C.c_int32), ("dim", C.c_int32), ("nen", C.c_int32),
                ("ndpn", C.c_int32), ("ngp", C.c_int32), ("structured", C.c_int32),
                ("n_nodes", C.c_int64), ("n_elems", C.c_int64), ("n_owned_nodes", C.c_int64),
                ("n_rows", C.c_int64), ("nnz", C.c_int64), ("nx", C.c_int64), ("ny", C.c_int64),
                ("nz", C.c_int64), ("device_bytes", C.c_int64)]


_lib = None


def load() -> C.CDLL:
    """Load liblgdm.so (built by ``__graft_entry__.build()``); raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, dp, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_int64
    L.lgdm_create_mesh.argtypes = [C.c_int, i64, vp, i64, vp, C.POINTER(Material), i64, i64, i64,
                                   i64, C.c_int, vp, C.POINTER(vp)]
    L.lgdm_set_state.argtypes = [vp, vp, i64, vp, i64, C.c_int]
    L.lgdm_assemble.argtypes = [vp, C.POINTER(CSR), C.POINTER(vp)]
    L.lgdm_update_history.argtypes = [vp]
    L.lgdm_residual_sumsq.argtypes = [vp, vp, C.c_int]
    L.lgdm_residual_norms.argtypes = [vp, dp]
    L.lgdm_set_comm.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
    L.lgdm_nccl_unique_id.argtypes = [vp, i64]
    L.lgdm_get_kappa.argtypes = [vp, vp]
    L.lgdm_scale_dofs.argtypes = [vp, C.c_double]
    L.lgdm_set_kernel.argtypes = [vp, C.c_int]
    L.lgdm_get_info.argtypes = [vp, C.POINTER(Info)]
    L.lgdm_launch_count.argtypes = [vp]
    L.lgdm_launch_count.restype = C.c_int64
    L.lgdm_last_error.restype = C.c_char_p
    L.lgdm_destroy.argtypes = [vp]
    L.lgdm_sdv_width.argtypes = [C.c_int]
    L.lgdm_set_defects.argtypes = [vp, vp, vp, i64, C.c_int]
    L.lgdm_update_state.argtypes = [vp, vp, i64, C.c_int]
    L.lgdm_get_blocked.argtypes = [vp, C.POINTER(CSR), C.POINTER(vp)]
    L.lgdm_apply_dirichlet.argtypes = [vp, i64, vp, vp]
    L.lgdm_solve.argtypes = [vp, vp, C.c_double, C.c_int, C.POINTER(C.c_int), dp]
    L.lgdm_add_dofs.argtypes = [vp, vp, C.c_double]
    L.lgdm_delta_norms.argtypes = [vp, vp, dp]
    L.lgdm_delta_ratios.argtypes = [vp, vp, C.c_double, dp, C.POINTER(C.c_int)]
    L.lgdm_step.argtypes = [vp, C.c_int, dp]
    L.lgdm_reaction.argtypes = [vp, i64, vp, dp]
    L.lgdm_solve_direct.argtypes = [vp, vp, C.POINTER(C.c_int)]
    L.lgdm_dof_offsets.argtypes = [vp, vp, i64]
    L.lgdm_create_mesh_mixed.argtypes = [C.c_int, i64, vp, i64, vp, C.POINTER(Material), i64, i64,
                                         i64, i64, i64, i64, C.c_int, vp, C.POINTER(vp)]
    L.lgdm_prefetch_dofs.argtypes = [vp, vp, i64]
    L.lgdm_set_state_prefetched.argtypes = [vp]
    for name in EXPORTS:
        if name not in ("lgdm_launch_count", "lgdm_last_error", "lgdm_destroy"):
            getattr(L, name).restype = C.c_int
    L.lgdm_destroy.restype = None
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise LGDMError(status, load().lgdm_last_error().decode())


def material(**kw) -> Material:
    """Material from keyword arguments (``t`` is accepted for ``thickness_or_area``)."""
    m = Material()
    for k, v in kw.items():
        setattr(m, "thickness_or_area" if k == "t" else k, v)
    return m


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for lgdm_set_comm; call on rank 0 and broadcast."""
    buf = C.create_string_buffer(128)
    _check(load().lgdm_nccl_unique_id(buf, 128))
    return buf.raw


class DeviceArray:
    """Zero-copy view of mesh-owned device memory (``torch.as_tensor(x, device='cuda')``)."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self._owner = owner
        # "stream": consumers (torch.as_tensor, CuPy) order their first use after the work
        # enqueued on the mesh's stream (CUDA Array Interface v3; 1 = the legacy default stream)
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None,
                                         "stream": int(getattr(owner, "stream", 0) or 1)}

    def torch(self, device=None):
        import torch
        return torch.as_tensor(self, device=device or "cuda")


def _ptr_and_kind(x):
    """(pointer, on_device, keepalive) of a float64 contiguous numpy array or torch tensor."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            assert x.dtype == torch.float64 and x.is_contiguous(), "need contiguous float64"
            return x.data_ptr(), 1 if x.is_cuda else 0, x
    except ImportError:
        pass
    a = np.ascontiguousarray(x, dtype=np.float64)
    return a.ctypes.data, 0, a


def _numel(x) -> int:
    """Element count of the caller's buffer (what the library's size checks compare)."""
    n = getattr(x, "numel", None)
    return int(n()) if callable(n) else int(np.asarray(x).size)


def _device_vector(x, n: int, device: int, what: str):
    """Validate a device float64 vector of n entries on the mesh's device."""
    import torch
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()):
        raise ValueError(f"{what}: need a contiguous float64 CUDA tensor")
    if x.numel() != n or x.device.index != device:
        raise ValueError(f"{what}: need {n} entries on cuda:{device}, got {x.numel()} on {x.device}")
    return x.data_ptr()


class Mesh:
    """One mesh (whole or one rank's slab) on one GPU.  See include/lgdm.h."""

    def __init__(self, etype: int, coords, conn, mat: Material, global_node_offset: int = 0,
                 n_global_nodes: int | None = None, owned=None, device: int = 0, stream=None,
                 global_dof_offset: int | None = None, n_global_dofs: int | None = None):
        L = load()
        self.etype = etype
        self.dim, self.nen, self.ndpn, self.ngp = FAMILY[etype]
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        conn = np.ascontiguousarray(conn, dtype=np.int64)
        self.n_nodes, self.n_elems = coords.shape[0], conn.shape[0]
        if n_global_nodes is None:
            n_global_nodes = global_node_offset + self.n_nodes
        owned = (0, self.n_nodes) if owned is None else owned
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(device).cuda_stream
        self.device = device
        self.stream = int(stream or 0)
        self.nranks, self.rank = 1, 0
        self._h = C.c_void_p()
        if global_dof_offset is not None:          # mixed-order slab
            _check(L.lgdm_create_mesh_mixed(etype, self.n_nodes, coords.ctypes.data, self.n_elems,
                                            conn.ctypes.data, C.byref(mat), global_node_offset,
                                            n_global_nodes, owned[0], owned[1], global_dof_offset,
                                            -1 if n_global_dofs is None else n_global_dofs,
                                            device, stream, C.byref(self._h)))
        else:
            _check(L.lgdm_create_mesh(etype, self.n_nodes, coords.ctypes.data, self.n_elems,
                                      conn.ctypes.data, C.byref(mat), global_node_offset,
                                      n_global_nodes, owned[0], owned[1], device, stream,
                                      C.byref(self._h)))
        self._keep = []
        self.doff = np.zeros(self.n_nodes + 1, dtype=np.int64)
        _check(L.lgdm_dof_offsets(self._h, self.doff.ctypes.data, self.doff.size))
        self.n_dofs = int(self.doff[-1])

    # -- state / assembly -------------------------------------------------------------
    def set_state(self, dofs, kappa=None):
        pd, on_dev, kd = _ptr_and_kind(dofs)
        if kappa is None:
            _check(load().lgdm_set_state(self._h, pd, _numel(kd), None, 0, on_dev))
            self._keep = [kd]
            return
        pk, on_dev_k, kk = _ptr_and_kind(kappa)
        if on_dev_k != on_dev:
            raise ValueError("dofs and kappa must both be host or both be device")
        _check(load().lgdm_set_state(self._h, pd, _numel(kd), pk, _numel(kk), on_dev))
        self._keep = [kd, kk]   # host copies are async only for pinned memory; keep alive

    def prefetch_dofs(self, dofs):
        """Start copying the next iterate's dofs (pinned host tensor / array) on the mesh's copy
        stream, overlapped with the work already enqueued (include/lgdm.h)."""
        p, on_dev, keep = _ptr_and_kind(dofs)
        if on_dev:
            raise ValueError("prefetch_dofs takes host memory")
        # the library double-buffers: the previous buffer may still be in flight, keep both
        self._keep_prefetch = (getattr(self, "_keep_prefetch", (None, None))[1], keep)
        _check(load().lgdm_prefetch_dofs(self._h, p, _numel(keep)))

    def set_state_prefetched(self):
        _check(load().lgdm_set_state_prefetched(self._h))

    def assemble(self):
        """Returns (row_ptr, col_idx, val, R, first_row, n_cols) as zero-copy device views."""
        csr = CSR()
        r = C.c_void_p()
        _check(load().lgdm_assemble(self._h, C.byref(csr), C.byref(r)))
        self.csr = csr
        return dict(row_ptr=DeviceArray(csr.row_ptr, csr.n_rows + 1, "<i8", self),
                    col_idx=DeviceArray(csr.col_idx, csr.nnz, "<i4", self),
                    val=DeviceArray(csr.val, csr.nnz, "<f8", self),
                    R=DeviceArray(r.value, csr.n_rows, "<f8", self),
                    first_row=csr.first_row, n_cols=csr.n_cols, n_rows=csr.n_rows, nnz=csr.nnz)

    # -- Newton loop pieces --------------------------------------------
    def apply_dirichlet(self, dof_ids, increments):
        ids = np.ascontiguousarray(dof_ids, dtype=np.int64)
        inc = np.ascontiguousarray(increments, dtype=np.float64)
        _check(load().lgdm_apply_dirichlet(self._h, ids.size, ids.ctypes.data if ids.size else None,
                                           inc.ctypes.data if inc.size else None))

    def solve(self, tol=1e-12, max_iter=10000, out=None):
        """BiCGSTAB on the assembled (eliminated) system; returns (delta device tensor, iters,
        relative residual)."""
        import torch
        n = self.n_dofs
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")
        it = C.c_int()
        rr = C.c_double()
        _check(load().lgdm_solve(self._h, out.data_ptr(), tol, max_iter, C.byref(it), C.byref(rr)))
        return out, it.value, rr.value

    def solve_direct(self, out=None):
        """Sparse QR on the GPU (cuSOLVER); returns the delta device tensor."""
        import torch
        n = self.n_dofs
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")
        sing = C.c_int()
        _check(load().lgdm_solve_direct(self._h, out.data_ptr(), C.byref(sing)))
        return out

    def reaction(self, dof_ids):
        ids = np.ascontiguousarray(dof_ids, dtype=np.int64)
        out = C.c_double()
        _check(load().lgdm_reaction(self._h, ids.size, ids.ctypes.data if ids.size else None,
                                    C.byref(out)))
        return out.value

    def add_dofs(self, delta, alpha=1.0):
        p = _device_vector(delta, self.n_dofs, self.device, "add_dofs")
        _check(load().lgdm_add_dofs(self._h, p, alpha))

    def delta_norms(self, delta):
        p = _device_vector(delta, self.n_dofs, self.device, "delta_norms")
        out = np.zeros(4)
        _check(load().lgdm_delta_norms(self._h, p, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def converged(self, delta, tol):
        """Alg. 1 l.26 / Alg. 2 l.16 convergence test in the library: returns
        (converged, |du|/|u|, |de|/|e|) for the correction delta (lgdm_delta_ratios)."""
        p = _device_vector(delta, self.n_dofs, self.device, "converged")
        out = np.zeros(2)
        flag = C.c_int()
        _check(load().lgdm_delta_ratios(self._h, p, tol, out.ctypes.data_as(C.POINTER(C.c_double)),
                                        C.byref(flag)))
        return bool(flag.value), float(out[0]), float(out[1])

    def get_blocked(self):
        """K, R of the last assemble in the blocked DOF order [u; ebar] (zero-copy views)."""
        csr = CSR()
        r = C.c_void_p()
        _check(load().lgdm_get_blocked(self._h, C.byref(csr), C.byref(r)))
        return dict(row_ptr=DeviceArray(csr.row_ptr, csr.n_rows + 1, "<i8", self),
                    col_idx=DeviceArray(csr.col_idx, csr.nnz, "<i4", self),
                    val=DeviceArray(csr.val, csr.nnz, "<f8", self),
                    R=DeviceArray(r.value, csr.n_rows, "<f8", self),
                    n_rows=csr.n_rows, nnz=csr.nnz)

    def set_defects(self, kappa0_gp=None, alpha_gp=None):
        """Per-GP kappa0 / alpha ([n_elems, ngp] or flat; None = material value)."""
        n = None
        ptrs, keep, dev = [], [], None
        for a in (kappa0_gp, alpha_gp):
            if a is None:
                ptrs.append(None)
                continue
            p, on_dev, k = _ptr_and_kind(a)
            if dev is not None and dev != on_dev:
                raise ValueError("kappa0_gp and alpha_gp must both be host or both be device")
            if n is not None and _numel(k) != n:
                raise ValueError("kappa0_gp and alpha_gp must have the same size")
            dev = on_dev
            n = _numel(k)
            ptrs.append(p)
            keep.append(k)
        _check(load().lgdm_set_defects(self._h, ptrs[0], ptrs[1], n or 0, dev or 0))
        self._keep_defects = keep

    def update_state(self, out=None):
        """State-variable update (Alg. 2 l.8-14) + history commit.  Returns a device tensor
        [n_elems, ngp, sdv_width] (or fills `out`, a float64 tensor / numpy array)."""
        import torch
        W = load().lgdm_sdv_width(self.etype)
        if W < 0:
            raise LGDMError(1, f"element type {self.etype} has no state record")
        if out is None:
            out = torch.empty((self.n_elems, self.ngp, W), dtype=torch.float64,
                              device=f"cuda:{self.device}")
        p, on_dev, keep = _ptr_and_kind(out)
        _check(load().lgdm_update_state(self._h, p, _numel(keep), on_dev))
        return out

    def update_history(self):
        _check(load().lgdm_update_history(self._h))

    def residual_sumsq(self, out_device_ptr: int | None = None):
        """Device-side (stream-ordered) if a device pointer is given, else returns host [2]."""
        if out_device_ptr is not None:
            _check(load().lgdm_residual_sumsq(self._h, out_device_ptr, 1))
            return None
        out = np.zeros(2)
        _check(load().lgdm_residual_sumsq(self._h, out.ctypes.data, 0))
        return out

    def step(self, graph: bool = True, history: bool = False):
        """One hot-path pass (lgdm_step): assemble, residual norms (allreduce across ranks),
        optionally the history commit; CUDA-graph replay after the first call.  Returns the
        norms {||Fu||, ||Fe||}."""
        out = np.zeros(2)
        _check(load().lgdm_step(self._h, (1 if graph else 0) | (2 if history else 0),
                                out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def residual_norms(self):
        out = np.zeros(2)
        _check(load().lgdm_residual_norms(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_comm(self, unique_id: bytes, nranks: int, rank: int):
        _check(load().lgdm_set_comm(self._h, unique_id, nranks, rank))
        self.nranks, self.rank = nranks, rank

    def get_kappa(self):
        out = np.zeros((self.n_elems, self.ngp))
        _check(load().lgdm_get_kappa(self._h, out.ctypes.data))
        return out

    def scale_dofs(self, s: float):
        _check(load().lgdm_scale_dofs(self._h, s))

    def set_kernel(self, kernel: int):
        _check(load().lgdm_set_kernel(self._h, kernel))

    def info(self) -> dict:
        inf = Info()
        _check(load().lgdm_get_info(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in Info._fields_}

    @property
    def launches(self) -> int:
        return int(load().lgdm_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().lgdm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sdv_width(etype: int) -> int:
    """doubles per (element, GP) record of Mesh.update_state (include/lgdm.h)"""
    return load().lgdm_sdv_width(etype)


def newton(mesh: "Mesh", fixed_dofs, step_increment, n_steps: int, tol: float = 1e-4,
           max_iter: int = 25, solver_tol: float = 1e-10, solver: str = "direct"):
    """Incremental-iterative Newton driver of Alg. 2 (orchestration only --
    every computation is a library call on the GPU): for each of n_steps load steps, iterate
    assemble (trial kappa against the committed history) -> eliminate the constraints
    (increment on the first iteration, 0 after) -> solve (sparse QR on the GPU as the paper's
    mldivide, or solver="bicgstab") -> dofs += delta until
    ||du||/||u|| and ||de||/||e|| <= tol (Alg. 2 l.16), then record the reaction at the driven
    dofs (nonzero increments) and commit the history.  Returns one dict per step (iterations,
    final ratios, solver iterations, reaction).  Raises LGDMError if a step does
    not converge in max_iter iterations."""
    if solver == "direct" and getattr(mesh, "nranks", 1) > 1:
        solver = "bicgstab"                   # the sparse QR is single-rank; Krylov across slabs
    fixed = np.ascontiguousarray(fixed_dofs, dtype=np.int64)
    inc = np.broadcast_to(np.asarray(step_increment, dtype=np.float64), fixed.shape).copy()
    zero = np.zeros_like(inc)
    log = []
    driven = fixed[inc != 0.0]
    for step in range(n_steps):
        for it in range(1, max_iter + 1):
            mesh.assemble()
            mesh.apply_dirichlet(fixed, inc if it == 1 else zero)
            if solver == "direct":
                delta, sit, rr = mesh.solve_direct(), 0, 0.0
            else:
                delta, sit, rr = mesh.solve(tol=solver_tol)
            mesh.add_dofs(delta)
            done, ru, re = mesh.converged(delta, tol)
            if done:
                break
        else:
            raise LGDMError(8, f"Newton step {step}: not converged in {max_iter} iterations "
                               f"(|du|/|u| = {ru:.3e}, |de|/|e| = {re:.3e})")
        mesh.assemble()                       # converged state: reaction at the driven dofs
        react = mesh.reaction(driven)
        mesh.update_history()
        log.append(dict(step=step, iterations=it, ratio_u=ru, ratio_e=re, solver_iters=sit,
                        solver_relres=rr, reaction=react))
    return log
