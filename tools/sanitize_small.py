"""Small assemblies of every structured kernel (for compute-sanitizer runs)."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import synth
from paper_2301_06503_b200 import lgdm
from parity import gpu_assemble
cases = [(lgdm.QUAD4, (40, 5), 4), (lgdm.HEX8, (5, 9, 3), 4), (lgdm.HEX8, (5, 9, 3), 5)]
for et, n, k in cases:
    cfg = synth.small_config(et, n)
    mesh = synth.structured_mesh(cfg)
    d, kap = synth.fields(cfg, mesh)
    gpu_assemble(et, mesh.coords, mesh.conn, d, kap, kernel=k)
    print('done', et, n, k, flush=True)
