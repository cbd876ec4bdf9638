"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the structured sweeps (k_sweepq, k_sweep4), the general path, the mixed-order
kernels, the state update, the history update, the norms and the A0 pattern build.
usage: compute-sanitizer --tool <tool> python tools/sanitize_small.py
(compute-sanitizer is closed on this pool -- it refuses to run; the substitutes are the
bitwise-reproducibility and slab-stitching tests and the parity suite.)"""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import synth
from paper_2301_06503_b200 import lgdm

MAT = lgdm.material(**synth.MATERIAL)
cases = [(lgdm.QUAD4, (40, 5), lgdm.KERNEL_SWEEP), (lgdm.HEX8, (5, 9, 3), lgdm.KERNEL_SWEEP),
         (lgdm.QUAD4, (7, 6), lgdm.KERNEL_GENERAL), (lgdm.HEX8, (3, 4, 2), lgdm.KERNEL_GENERAL)]
for et, n, k in cases:
    cfg = synth.small_config(et, n)
    mesh = synth.structured_mesh(cfg)
    d, kap = synth.fields(cfg, mesh)
    m = lgdm.Mesh(et, mesh.coords, mesh.conn, MAT, stream=0)
    m.set_kernel(k)
    m.set_state(d, kap)
    m.assemble()
    m.residual_norms()
    m.update_state()
    m.update_history()
    m.close()
    print('done', et, n, k, flush=True)
mm = synth.mixed_mesh(synth.QUAD8, (6, 5))
d, kap = synth.mixed_fields(mm)
m = lgdm.Mesh(synth.QUAD8, mm.coords, mm.conn, MAT, stream=0)
m.set_state(d, kap)
m.assemble()
m.residual_norms()
m.update_state()
m.close()
print('done quad8', flush=True)
