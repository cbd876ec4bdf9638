"""The seeded input generator: determinism and slab invariance (global-id keying)."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("etype,n,layers", [(1, (12,), (3, 9)), (2, (7, 9), (2, 6)), (3, (4, 3, 6), (1, 4))])
def test_slab_matches_full(etype, n, layers):
    cfg = synth.small_config(etype, n)
    full = synth.structured_mesh(cfg)
    fd, fk = synth.fields(cfg, full)
    slab = synth.structured_mesh(cfg, elem_layers=layers)
    sd, sk = synth.fields(cfg, slab)
    g = slab.node_gid0 + np.arange(slab.coords.shape[0])
    np.testing.assert_array_equal(slab.coords, full.coords[g])
    np.testing.assert_array_equal(sd, fd[g])
    np.testing.assert_array_equal(sk, fk[slab.elem_gid])
    np.testing.assert_array_equal(slab.conn + slab.node_gid0, full.conn[slab.elem_gid])


def test_structured_sizes_and_orientation():
    for cid in (0, 1):
        cfg = synth.CONFIGS[cid]
        m = synth.structured_mesh(cfg)
        assert m.coords.shape[0] == cfg.n_nodes and m.conn.shape[0] == cfg.n_elems
    cfg = synth.small_config(3, (2, 2, 2))
    m = synth.structured_mesh(cfg)
    X = m.coords[m.conn[0]]
    ref = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]])
    np.testing.assert_array_equal(X / cfg.h_el, ref)       # SURVEY 8c.1 local node order


def test_rng_determinism_and_moments():
    u = synth.uniform(1, 0, np.arange(200000, dtype=np.uint64))
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.005
    z = synth.normal(1, 2, np.arange(200000, dtype=np.uint64))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    np.testing.assert_array_equal(u, synth.uniform(1, 0, np.arange(200000, dtype=np.uint64)))


def test_branch_mix_config1():
    """The config-1 inputs exercise loading and unloading GPs (SURVEY 8c.5 branch mix)."""
    cfg = synth.CONFIGS[1]
    m = synth.structured_mesh(cfg)
    d, k = synth.fields(cfg, m)
    ebar_el = d[m.conn, 2].mean(axis=1)
    frac_loading = (ebar_el[:, None] > k).mean()
    assert 0.3 < frac_loading < 0.9
    assert (k == 1e-4).mean() == pytest.approx(0.25, abs=0.01)
