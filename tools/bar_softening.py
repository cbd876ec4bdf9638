"""1D bar softening run through the GPU Newton loop (the paper's §3.1 setting
with equal-order elements): defect region in the middle (lower kappa0), displacement control."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import synth
from paper_2301_06503_b200 import lgdm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
umax = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
cfg = synth.small_config(lgdm.BAR2, (n,))
mesh = synth.structured_mesh(cfg)
L = mesh.coords[-1, 0] - mesh.coords[0, 0]
mat = dict(synth.MATERIAL)
m = lgdm.Mesh(lgdm.BAR2, mesh.coords, mesh.conn, lgdm.material(**mat))
m.set_state(np.zeros(2 * (n + 1)), np.zeros(2 * n))
xc = mesh.coords[mesh.conn, 0].mean(axis=1)
k0 = np.where(np.abs(xc - (mesh.coords[0, 0] + L / 2)) < 0.05 * L, 0.9, 1.0) * mat["kappa0"]
m.set_defects(np.repeat(k0, 2), None)
t0 = time.time()
log = lgdm.newton(m, [0, 2 * n], [0.0, umax / steps], n_steps=steps, tol=1e-6, max_iter=40)
r = np.array([s["reaction"] for s in log])
print("time", time.time() - t0, "iters", [s["iterations"] for s in log][:20], "max solver its",
      max(s["solver_iters"] for s in log))
ip = int(r.argmax())
print("peak", r.max(), "at step", ip, "final", r[-1], "final/peak", r[-1] / r.max())
print("reactions", np.round(r[::max(1, steps // 20)], 4))
