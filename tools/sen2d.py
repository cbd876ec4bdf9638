"""2D side-edge-notch (SEN) run with the paper's own 2D discretisation (QUAD8 serendipity u,
bilinear ebar) through the GPU Newton loop: SPEC default geometry (100 x 100 mm plate,
50 mm mid-height edge slit), bottom edge fixed, top edge pulled in y (displacement control).
Reading R2 (h_sigma = 0: Eq. 11a and Fig. 2 line 19 literally): with R1
the Hessian of the equivalent strain, unbounded as the strain goes to zero (the flanks of the
slit), makes full Newton cycle on fine meshes -- in the oracle as well.
Reports the load-displacement curve, where damage starts and the damage band."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2301_06503_b200 import lgdm  # noqa: E402


def run(n=50, steps=60, du=5e-4, tol=1e-5, verbose=True):
    mesh = synth.sen_mesh(synth.QUAD8, (n, n))
    X = mesh.coords
    mat = dict(synth.MATERIAL, h_sigma=0.0)
    m = lgdm.Mesh(lgdm.QUAD8, X, mesh.conn, lgdm.material(**mat))
    doff = m.doff
    # bottom edge: u_y = 0, u_x = 0 at the bottom-left corner only; top edge: u_y = delta
    bot = np.nonzero(X[:, 1] < 1e-9)[0]
    top = np.nonzero(X[:, 1] > X[:, 1].max() - 1e-9)[0]
    corner = bot[np.argmin(X[bot, 0])]
    ids = np.concatenate([[doff[corner]], doff[bot] + 1, doff[top] + 1])
    inc = np.concatenate([[0.0], np.zeros(bot.size), np.full(top.size, du)])
    ne = mesh.conn.shape[0]
    m.set_state(np.zeros(m.n_dofs), np.zeros((ne, 9)))
    t0 = time.time()
    log, first = [], None
    centres = X[mesh.conn[:, :4]].mean(axis=1)
    for st in range(steps):
        log += lgdm.newton(m, ids, inc, n_steps=1, tol=tol, max_iter=60)
        if first is None:
            k = m.get_kappa().max(axis=1)
            if k.max() > synth.MATERIAL["kappa0"]:
                first = (st, centres[int(k.argmax())])
    r = np.array([s["reaction"] for s in log])
    kap = m.get_kappa()
    if verbose and first is not None:
        print("damage starts at step", first[0], "in the element centred at", np.round(first[1], 2))
    if verbose:
        print(f"SEN {n}x{n}: {steps} steps in {time.time() - t0:.1f} s, iterations "
              f"{[s['iterations'] for s in log]}")
        print("reaction", np.round(r, 3))
    return mesh, log, r, kap


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    du = float(sys.argv[3]) if len(sys.argv) > 3 else 5e-4
    tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-5
    mesh, log, r, kap = run(n, steps, du, tol)
    X = mesh.coords
    c = X[mesh.conn[:, :4]].mean(axis=1)
    k = kap.max(axis=1)
    print("peak", r.max(), "at step", int(r.argmax()), "final/peak", r[-1] / r.max())
    top = np.argsort(k)[-5:]
    print("most damaged element centres", np.round(c[top], 2))
