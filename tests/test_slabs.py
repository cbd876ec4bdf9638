"""Host logic of the slab partition (CPU)."""
import numpy as np
import pytest

import synth
from paper_2301_06503_b200 import slabs


@pytest.mark.parametrize("n,P", [((10,), 3), ((5, 8), 4), ((4, 3, 6), 7), ((3, 3, 200), 8), ((2, 2, 1), 2)])
def test_slabs_cover_each_node_once(n, P):
    L = n[-1]
    owned = []
    for p in range(P):
        s = slabs.slab(n, p, P)
        b, e = s.owned_nodes
        assert e > b
        owned.append((b, e))
        lb, le = s.local_nodes
        assert lb <= b and e <= le
        # every element touching an owned node is local
        assert s.elem_layers[0] <= max(s.node_layers[0] - 1, 0)
        assert s.elem_layers[1] >= min(s.node_layers[1], L)
    flat = np.concatenate([np.arange(b, e) for b, e in owned])
    total = int(np.prod([k + 1 for k in n]))
    np.testing.assert_array_equal(flat, np.arange(total))


def test_slab_mesh_ranges_match_generator():
    cfg = synth.small_config(3, (3, 4, 9))
    for p in range(4):
        s = slabs.slab(cfg.n, p, 4)
        m = synth.structured_mesh(cfg, elem_layers=s.elem_layers)
        assert m.node_gid0 == s.local_nodes[0]
        assert m.node_gid0 + m.coords.shape[0] == s.local_nodes[1]
        ob, oe = s.owned_local(m.node_gid0)
        assert 0 <= ob < oe <= m.coords.shape[0]


def test_recompute_overhead_config4():
    per = slabs.elements_per_rank((200, 200, 200), 8)
    assert sum(per) <= 1.08 * 8_000_000 and max(per) <= 1.08 * 1_000_000
