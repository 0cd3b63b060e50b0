"""Per-CUDA-source-line executed instructions and stall samples: tools/ncu_lines.py <rep> [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; agg = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = r; continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        agg.append((fname, r[0], r[1], float(r[hdr.index('Instructions Executed')] or 0), float(r[hdr.index('# Samples')] or 0)))
    except ValueError:
        pass
T = sum(a[3] for a in agg) or 1; S = sum(a[4] for a in agg) or 1
for f, ln, src, ex, sm in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{ex/T*100:5.1f}% ex {sm/S*100:5.1f}% smp {f}:{ln} {src.strip()[:90]}")
