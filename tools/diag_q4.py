"""Debug helper: which nodes of a Q4 mesh disagree with the oracle (the sweep kernel)."""
import sys
import numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import synth, oracle
from paper_2301_06503_b200 import lgdm
from parity import gpu_assemble
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = synth.CONFIGS[cid]
mesh = synth.structured_mesh(cfg)
d, k = synth.fields(cfg, mesh)
ref = oracle.assemble(cfg.etype, oracle.material(**synth.MATERIAL), mesh.coords, mesh.conn, d, k)
got = gpu_assemble(cfg.etype, mesh.coords, mesh.conn, d, k, kernel=lgdm.KERNEL_SWEEP)
rp = ref['row_ptr']; nrows = rp.size - 1
rows = np.repeat(np.arange(nrows), np.diff(rp))
rowmax = np.zeros(nrows); np.maximum.at(rowmax, rows, np.abs(ref['val']))
bad = np.abs(got['val'] - ref['val']) > 1e-12 * rowmax[rows]
nx = cfg.n[0] + 1
bn = np.unique(rows[bad] // 3)
print('bad entries', bad.sum(), 'bad nodes', bn.size)
print('nodes (x,y):', [(int(n % nx), int(n // nx)) for n in bn[:40]])
ys = np.unique(bn // nx); xs = np.unique(bn % nx)
print('rows y:', ys[:60]); print('cols x:', xs[:60])
ci = ref['col_idx']
same = (ci[bad] // 3) == rows[bad] // 3
print('fraction of bad entries in the diagonal block:', same.mean() if bad.any() else 0)
dr = np.abs(got['R'] - ref['R']) > 1e-12 * ref['S']
print('bad R rows', dr.sum(), [(int(r // 3 % nx), int(r // 3 // nx), int(r % 3)) for r in np.nonzero(dr)[0][:20]])
