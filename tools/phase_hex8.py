"""Per-phase cycle breakdown of k_hex8 (debug build gpurun_out/lib_timing.so,
-DLGDM_PHASE_TIMING): thread 0 of the PC, TW and MW roles accumulate clock64 deltas."""
import ctypes as C
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LGDM_LIB"] = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "lib_timing.so")
import torch
import synth
from paper_2301_06503_b200 import lgdm
L = lgdm.load()
L.lgdm_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
names = {0: "C wait core-full", 1: "C tiles+expansions (rnd 0) / expansions", 2: "C moments",
         3: "C reduce+picks+ns", 4: "C colour barrier", 5: "C adds", 6: "C end-layer barrier",
         7: "C flush", 8: "C reset barrier", 9: "C batch prologue", 10: "PC wait core-empty",
         11: "PC core", 12: "PC other", 15: "PC wait adds-done", 14: "PC flush"}
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.CONFIGS[cid]
mesh = synth.structured_mesh(cfg)
d, k = synth.fields(cfg, mesh)
m = lgdm.Mesh(cfg.etype, mesh.coords, mesh.conn, lgdm.material(**synth.MATERIAL))
m.set_kernel(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
m.set_state(d, k)
m.assemble(); torch.cuda.synchronize()
buf = np.zeros(16, dtype=np.uint64)
L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
m.assemble(); torch.cuda.synchronize()
L.lgdm_debug_phase_cycles(buf.ctypes.data, 1)
for grp in ("PC", "C"):
    idx = [i for i, n in names.items() if n.startswith(grp + " ")]
    tot = float(sum(buf[i] for i in idx))
    print(cfg.name, grp, "total %.4e cycles (sum over CTAs of thread 0)" % tot)
    for i in idx:
        print(f"  {names[i]:24s} {float(buf[i]):.3e}  {100 * float(buf[i]) / max(tot, 1):5.1f}%")
