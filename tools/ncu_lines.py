"""Aggregate ncu source-page stall samples per CUDA source line (needs -lineinfo)."""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur = None
    agg = []
    tot = 0.0
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] not in ('',):
            try:
                w = float(r[4])
                n = float(r[7])
            except ValueError:
                continue
            agg.append((w, cur, r[0], r[1][:100], n))
            tot += w
    agg.sort(reverse=True)
    print('total stall samples', tot)
    for w, f, l, s, n in agg[:top]:
        print(f'{100 * w / tot:5.1f}%  {f}:{l:<5} inst={n:>12.0f}  {s}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
