"""Shared-memory wavefronts per CUDA source line of an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; agg = []; tot = 0
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr and r and r[0] and len(r) > 20:
        try: wf = float(r[hdr['L1 Wavefronts Shared']]); ideal = float(r[hdr.get('L1 Wavefronts Shared Ideal', hdr['L1 Wavefronts Shared'])])
        except (ValueError, KeyError): continue
        if wf > 0: agg.append((wf, ideal, cur, r[0], r[1][:80])); tot += wf
agg.sort(reverse=True)
print('total', tot)
for wf, ideal, f, l, s in agg[:30]: print(f'{100*wf/tot:5.1f}% (ideal {100*ideal/tot:5.1f}%) {f}:{l:<5} {s}')
