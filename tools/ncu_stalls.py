"""Stall-reason breakdown (share of warp samples) of an ncu report: tools/ncu_stalls.py <rep>"""
import csv, io, subprocess, sys
from collections import Counter
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]; data = rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith('stall_') and '(' not in h]
    tot = Counter()
    for row in data:
        for r in reasons:
            try:
                tot[r] += float(row[idx[r]] or 0)
            except (ValueError, IndexError):
                pass
    S = sum(tot.values()) or 1
    print(rep, ' '.join(f"{r[6:]}={v / S * 100:.0f}%" for r, v in tot.most_common(8)))
