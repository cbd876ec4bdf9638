"""Time lgdm_assemble for knock-out builds tools/liblgdm_exp*.so (diagnostics only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2301_06503_b200 import lgdm
lib = sys.argv[1]
lgdm.LIB_PATH = lib
for cid in [int(c) for c in sys.argv[2:]]:
    cfg = synth.CONFIGS[cid]
    mesh = synth.structured_mesh(cfg)
    d, k = synth.fields(cfg, mesh)
    m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(d, k)
    for _ in range(3): m.assemble()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): m.assemble()
    b.record(); torch.cuda.synchronize()
    print(os.path.basename(lib), cfg.name, round(a.elapsed_time(b) / 5, 3), "ms")
