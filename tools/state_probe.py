"""Run lgdm_update_state on a synthetic config (for ncu captures)."""
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
out = m.update_state()
for _ in range(3):
    m.update_state(out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    m.update_state(out=out)
e.record()
torch.cuda.synchronize()
print("update_state ms", s.elapsed_time(e) / 5)
