import sys
sys.path.insert(0, '.')
import numpy as np, synth
from paper_2301_06503_b200 import lgdm

cfg = synth.CONFIGS[1]                                   # Q4 200 x 200, plane strain
mesh = synth.structured_mesh(cfg)
dofs, kappa = synth.fields(cfg, mesh)
m = lgdm.Mesh(lgdm.QUAD4, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
m.set_state(dofs, kappa)
out = m.assemble()                     # device CSR K (row_ptr, col_idx, val) and R, zero-copy
K_val = out["val"].torch()             # torch view of the device values
un, ue = m.residual_norms()            # ||R_u||, ||R_e||
m.update_history()                     # commit kappa (Eq. A.2)
print("example ok", K_val.shape, un, ue)
