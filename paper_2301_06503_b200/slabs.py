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
