"""Debug: worst K entry of the QUAD8 bench-size parity."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch, oracle, synth
from paper_2301_06503_b200 import lgdm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
mesh = synth.mixed_mesh(5, (n, n), 100.0)
dofs, kap = synth.mixed_fields(mesh)
MAT = dict(synth.MATERIAL)
ref = oracle.mixed_assemble(5, oracle.material(**MAT), mesh.coords, mesh.conn, dofs, kap)
m = lgdm.Mesh(5, mesh.coords, mesh.conn, lgdm.material(**MAT)); m.set_state(dofs, kap)
out = m.assemble(); torch.cuda.synchronize()
val = out["val"].torch().cpu().numpy(); R = out["R"].torch().cpu().numpy()
rp = ref["row_ptr"]; rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
rowmax = np.zeros(rp.size - 1); np.maximum.at(rowmax, rows, np.abs(ref["val"]))
err = np.abs(val - ref["val"]) / rowmax[rows]
idx = np.argsort(err)[-8:]
kind = oracle.dof_kind(ref["doff"], 2)
node_of = np.repeat(np.arange(mesh.coords.shape[0]), np.diff(ref["doff"]))
for i in idx:
    r, c = rows[i], ref["col_idx"][i]
    print(f"err {err[i]:.3e} row {r} (node {node_of[r]} kind {kind[r]}) col {c} (node {node_of[c]} kind {kind[c]}) ref {ref["val"][i]:.17e} got {val[i]:.17e} rowmax {rowmax[r]:.3e}")
print("count > 1e-12:", (err > 1e-12).sum(), "of", err.size)
# elements of the worst entry's row node
r = rows[idx[-1]]; nd = node_of[r]
els = np.nonzero((mesh.conn == nd).any(axis=1))[0]
xi, _ = oracle.mixed_gauss(5)
for e in els:
    c = mesh.conn[e]
    Ng = np.array([oracle.mixed_shape(5, xi[g], "e")[0] for g in range(9)])
    eb = Ng @ np.array([dofs[ref["doff"][c[a]] + 2] for a in range(4)])
    print("elem", e, "kh", kap[e], "ebar_gp", eb, "ebar-kh", eb - kap[e])
