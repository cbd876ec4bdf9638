"""bench.py's JSON-line contract (task statement): the reference arm on the CPU, and the GPU arm
on a small configuration."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "1", "--steps", "3", "--warmup", "3", "--no-secondary"])
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0 < r["fp64"]["frac"] < 1 and r["attainable_frac"] >= max(r["frac"], r["fp64"]["frac"]) - 1e-12
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= c.keys()
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    assert d["config"]["workload"] == "q4_200x200"


def test_gpus_flag_launches_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks (rendezvous on
    127.0.0.1, gloo in --dry-run) and rank 0 reports n_gpus = 2."""
    d = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"], timeout=300)
    assert d["dry_run"] is True and d["n_gpus"] == 2 and d["ranks_joined"] == 2


def test_dofs_recipe():
    """dofs_t = (1 + 0.05 (t mod 10)) dofs_0: the per-step factors compose to the recipe."""
    sys.path.insert(0, ROOT)
    import bench
    f = 1.0
    for t in range(25):
        assert abs(f - (1 + 0.05 * (t % 10))) < 1e-12
        f *= bench.dofs_factor(t)


def test_cpu_colouring_is_race_free():
    """The 2^d colouring of the all-core CPU baseline: elements of one colour share no node."""
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    import synth
    for cid in (1, 3):
        cfg = synth.small_config(synth.CONFIGS[cid].etype, (5, 4) if cid == 1 else (5, 4, 3))
        mesh = synth.structured_mesh(cfg)
        col, nc = bench.structured_colours(cfg, mesh.conn.shape[0])
        for c in range(nc):
            nodes = mesh.conn[col == c].reshape(-1)
            assert nodes.size == np.unique(nodes).size
