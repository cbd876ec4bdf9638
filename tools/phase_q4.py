"""Per-phase cycle breakdown of k_sweepq (debug build lib_timing.so from tools/build_timing.sh):
thread 0 of the PC, C and flush roles accumulate clock64 deltas per phase."""
import ctypes as C
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LGDM_LIB"] = os.path.join(ROOT, "lib_timing.so")
import torch
import synth
from paper_2301_06503_b200 import lgdm
L = lgdm.load()
L.lgdm_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
names = {0: "C other", 1: "C wait slot-full", 2: "C stars (compute)", 3: "C wait add-order", 4: "C adds",
         14: "F wait adds", 5: "F diagonal", 6: "F barrier", 7: "F copy+R+edges", 8: "F ns reset", 9: "F other",
         12: "PC other", 10: "PC wait slot-empty", 11: "PC core+records"}
cfg = synth.CONFIGS[2]
mesh = synth.structured_mesh(cfg)
d, k = synth.fields(cfg, mesh)
m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
m.set_state(d, k)
m.assemble(); torch.cuda.synchronize()
buf = np.zeros(16, dtype=np.uint64)
L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
m.assemble(); torch.cuda.synchronize()
L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
for grp in ("C", "PC", "F"):
    idx = [i for i, n in names.items() if n.startswith(grp + " ")]
    tot = float(sum(buf[i] for i in idx))
    print(cfg.name, grp, "total %.4e cycles (sum over CTAs of thread 0)" % tot)
    for i in idx:
        print(f"  {names[i]:24s} {float(buf[i]):.3e}  {100 * float(buf[i]) / max(tot, 1):5.1f}%")
