"""Top SASS instructions by warp-stall samples: tools/ncu_hot.py <rep> [N]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and '(' not in h]
tot = sum(float(r[idx['# Samples']] or 0) for r in data)
ops = Counter()
for r in data:
    op = r[idx['Source']].strip().split()[0] if r[idx['Source']].strip() else '?'
    if op.startswith('@'):
        op = r[idx['Source']].strip().split()[1]
    ops[op.split('.')[0]] += float(r[idx['# Samples']] or 0)
print('samples by opcode:', ', '.join(f'{k}={v/tot*100:.1f}%' for k, v in ops.most_common(14)))
ex = Counter()
for r in data:
    op = r[idx['Source']].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith('@') else op[0]
    ex[o.split('.')[0]] += float(r[idx['Instructions Executed']] or 0)
T = sum(ex.values())
print('executed warp-instr by opcode:', ', '.join(f'{k}={v/T*100:.1f}%' for k, v in ex.most_common(14)), f'total={T:.3g}')
rows2 = sorted(data, key=lambda r: -float(r[idx['# Samples']] or 0))[:top]
for r in rows2:
    s = float(r[idx['# Samples']] or 0)
    st = sorted(((float(r[idx[x]] or 0), x[6:]) for x in reasons), reverse=True)[:3]
    print(f"{s/tot*100:5.2f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} " + ' '.join(f'{n}={v:.0f}' for v, n in st if v))
