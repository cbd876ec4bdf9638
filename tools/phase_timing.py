"""Per-phase cycle breakdown of k_sweep (debug build tools/liblgdm_timing.so)."""
import ctypes as C
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2301_06503_b200 import lgdm
lgdm.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblgdm_timing.so")
L = lgdm.load()
L.lgdm_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
names = ["PC: wait CEMPTY", "PC: core", "PE: wait CFULL", "PE: wait REMPTY", "PE: expand",
         "C: between GPs", "C: wait RFULL", "C: pair GP", "C: colour barrier", "C: smem add",
         "C: end-layer barrier", "C: flush+reset"]
for cid in [int(c) for c in sys.argv[1:]] or [3, 2]:
    cfg = synth.CONFIGS[cid]
    mesh = synth.structured_mesh(cfg)
    d, k = synth.fields(cfg, mesh)
    m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
    m.set_state(d, k)
    m.assemble()
    torch.cuda.synchronize()
    buf = np.zeros(16, dtype=np.uint64)
    L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
    m.assemble()
    torch.cuda.synchronize()
    L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
    for grp, idx in (("PC", [0, 1]), ("PE", [2, 3, 4]), ("C", [5, 6, 7, 8, 9, 10, 11])):
        tot = float(sum(buf[i] for i in idx))
        print(cfg.name, grp, "total %.3e cycles" % tot)
        for i in idx:
            print(f"  {names[i]:32s} {float(buf[i]):.3e}  {100*float(buf[i])/max(tot,1):5.1f}%")
