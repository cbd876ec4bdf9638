"""Row-owned slab partition of a structured mesh over ranks.

Rank p of P owns a contiguous range of node layers along the LAST axis (z for Hex8, y for
Q4, x for the bar) and assembles exactly those CSR rows.  It holds every element that
touches an owned node -- one ghost element layer per interior slab face -- and recomputes
those ghost elements, so K and R need no communication.  Columns are global dof ids, so the
rank CSRs are row slices of the one-GPU CSR (bitwise equal: the per-entry summation order
does not depend on the partition).  Only the residual norms are reduced across ranks.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    p: int
    P: int
    node_layers: tuple      # owned node layers [z0, z1)
    elem_layers: tuple      # local element layers [l0, l1) (owned + ghost)
    layer_nodes: int        # nodes per layer

    @property
    def owned_nodes(self):
        """Global node id range [begin, end) owned by this rank."""
        return (self.node_layers[0] * self.layer_nodes, self.node_layers[1] * self.layer_nodes)

    @property
    def local_nodes(self):
        """Global node id range of the local (owned + ghost) nodes."""
        return (self.elem_layers[0] * self.layer_nodes, (self.elem_layers[1] + 1) * self.layer_nodes)

    def owned_local(self, gid0: int):
        b, e = self.owned_nodes
        return (b - gid0, e - gid0)

    @property
    def n_elem_layers(self):
        return self.elem_layers[1] - self.elem_layers[0]


def split(total: int, P: int, p: int):
    """Balanced contiguous split of range(total) into P parts; part p."""
    q, r = divmod(total, P)
    b = p * q + min(p, r)
    return b, b + q + (1 if p < r else 0)


def slab(n: tuple, p: int, P: int) -> Slab:
    """Slab p of P for a structured mesh with element counts n (x fastest)."""
    L = n[-1]
    if not (1 <= P <= L + 1) or not (0 <= p < P):
        raise ValueError(f"cannot split {L + 1} node layers over {P} ranks")
    z0, z1 = split(L + 1, P, p)
    l0, l1 = max(z0 - 1, 0), min(z1, L)
    layer = 1
    for k in n[:-1]:
        layer *= k + 1
    return Slab(p, P, (z0, z1), (l0, l1), layer)


def elements_per_rank(n: tuple, P: int):
    """Computed elements per rank (owned + ghost) -- the recompute overhead."""
    per_layer = 1
    for k in n[:-1]:
        per_layer *= k
    return [slab(n, p, P).n_elem_layers * per_layer for p in range(P)]


# ---------------------------------------------------------------------------------------
# Mixed-order meshes (BAR3, QUAD8; lgdm_create_mesh_mixed): the half-spacing lattice of
# synth.mixed_mesh, numbered x-fastest by lattice rows (QUAD8: corner rows of 2 nx + 1 nodes
# and midside rows of nx + 1 nodes; BAR3: one node per lattice point).  Element row l spans
# lattice rows 2l .. 2l + 2.  A slab owns whole element-row boundaries: rank p owns lattice
# rows [2 B_p, 2 B_{p+1}) (the last rank also the top row), holds element rows
# [max(B_p - 1, 0), B_{p+1}) and so the contiguous node range of lattice rows
# [2 max(B_p - 1, 0), 2 B_{p+1}].
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class MixedSlab:
    node_range: tuple        # global node ids [begin, end) of the local nodes
    elem_range: tuple        # global element ids [begin, end) of the local elements
    owned_local: tuple       # owned local node range
    global_dof_offset: int   # global dof id of local dof 0
    n_global_dofs: int


def _mixed_rows(etype: int, n: tuple):
    """(nodes per lattice row, dofs per lattice row, element rows, elements per row)"""
    if etype == 5:   # QUAD8
        nx, ny = n
        nodes = [(2 * nx + 1) if j % 2 == 0 else (nx + 1) for j in range(2 * ny + 1)]
        dofs = [(3 * (nx + 1) + 2 * nx) if j % 2 == 0 else 2 * (nx + 1) for j in range(2 * ny + 1)]
        return nodes, dofs, ny, nx
    nel = n[0]       # BAR3: corners (2 dofs) at even lattice points, midsides (1 dof) at odd
    return [1] * (2 * nel + 1), [2 if j % 2 == 0 else 1 for j in range(2 * nel + 1)], nel, 1


def mixed_slab(etype: int, n: tuple, p: int, P: int) -> MixedSlab:
    nodes, dofs, rows, per = _mixed_rows(etype, n)
    if not (1 <= P <= rows) or not (0 <= p < P):
        raise ValueError(f"cannot split {rows} element rows over {P} ranks")
    ns, ds = [0], [0]
    for a, b in zip(nodes, dofs):
        ns.append(ns[-1] + a)
        ds.append(ds[-1] + b)
    b0, b1 = split(rows, P, p)
    l0 = max(b0 - 1, 0)
    top = min(2 * b1 + 1, len(nodes))
    nb, ne = ns[2 * l0], ns[top]
    ob = ns[2 * b0] - nb
    oe = (ns[2 * b1] if p < P - 1 else ns[-1]) - nb
    return MixedSlab((nb, ne), (l0 * per, b1 * per), (ob, oe), ds[2 * l0], ds[-1])
