"""One lgdm_assemble of a BASELINE config (for ncu captures of the assembly kernel).
usage: python tools/assemble_once.py [config=3] [kernel=0] [repeats=1]"""
import sys
sys.path.insert(0, '.')
import torch
import synth
from paper_2301_06503_b200 import lgdm
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = synth.CONFIGS[cid]
mesh = synth.structured_mesh(cfg)
d, k = synth.fields(cfg, mesh)
m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
if kernel:
    m.set_kernel(kernel)
m.set_state(d, k)
for _ in range(reps):
    m.assemble()
torch.cuda.synchronize()
print("assembled", cfg.name, "kernel", kernel)
