"""Aggregate ncu source-page metrics per CUDA source line (needs -lineinfo):
stall samples, instructions executed, shared-memory wavefronts."""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur = None
    hdr = None
    agg = []
    tot = {'stall': 0.0, 'inst': 0.0, 'wf': 0.0}
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = {k: i for i, k in enumerate(r) if k not in hdr_skip}
            continue
        if hdr and r and r[0] not in ('',) and len(r) > 20:
            try:
                st = float(r[hdr['Warp Stall Sampling (All Samples)']])
                ins = float(r[hdr['Instructions Executed']])
                wf = float(r[hdr['L1 Wavefronts Shared']])
            except (ValueError, KeyError):
                continue
            agg.append((st, cur, r[0], r[1][:90], ins, wf))
            tot['stall'] += st
            tot['inst'] += ins
            tot['wf'] += wf
    agg.sort(reverse=True)
    print('totals', tot)
    for st, f, l, s, ins, wf in agg[:top]:
        print(f'{100 * st / tot["stall"]:5.1f}% stall {100 * ins / tot["inst"]:5.1f}% inst '
              f'{100 * wf / max(tot["wf"], 1):5.1f}% smemwf  {f}:{l:<5} {s}')


hdr_skip = set()
if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def by_range(path, ranges):
    """ranges: {name: [(file, lo, hi), ...]} -> stall / inst / smem-wavefront shares"""
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr = None, None
    agg = {k: [0.0, 0.0, 0.0] for k in list(ranges) + ['other']}
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr and r and r[0] not in ('',) and len(r) > 20:
            try:
                ln = int(r[0])
                v = [float(r[hdr['Warp Stall Sampling (All Samples)']]), float(r[hdr['Instructions Executed']]),
                     float(r[hdr['L1 Wavefronts Shared']])]
            except (ValueError, KeyError):
                continue
            key = 'other'
            for k, rr in ranges.items():
                if any(cur == f and lo <= ln <= hi for f, lo, hi in rr):
                    key = k
                    break
            for i in range(3):
                agg[key][i] += v[i]
    tot = [sum(a[i] for a in agg.values()) for i in range(3)]
    for k, a in agg.items():
        print(f'{k:10s} stall {100*a[0]/tot[0]:5.1f}%  inst {100*a[1]/tot[1]:5.1f}%  smem-wf {100*a[2]/max(tot[2],1):5.1f}%')
