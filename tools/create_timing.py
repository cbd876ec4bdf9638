"""Wall time of lgdm_create_mesh for a BASELINE config (run with LGDM_CREATE_TIMING=1 for the
per-phase split printed by the library).  usage: python tools/create_timing.py [config=4]"""
import sys, time
sys.path.insert(0, '.')
import torch, synth
from paper_2301_06503_b200 import lgdm
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
t0 = time.time(); mesh = synth.structured_mesh(cfg); print("gen mesh", time.time() - t0, flush=True)
torch.cuda.init(); torch.cuda.synchronize()
for rep in range(2):
    t0 = time.time()
    m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    torch.cuda.synchronize()
    print("create", time.time() - t0, flush=True)
    m.close()
