"""One lgdm_assemble of a BASELINE config (for ncu captures of the assembly kernel)."""
import sys
sys.path.insert(0, '.')
import torch
import synth
from paper_2301_06503_b200 import lgdm
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.CONFIGS[cid]
mesh = synth.structured_mesh(cfg)
d, k = synth.fields(cfg, mesh)
m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
m.set_state(d, k)
m.assemble()
torch.cuda.synchronize()
print("assembled", cfg.name)
