"""Shared-memory wavefronts per SASS opcode from an ncu report: python tools/ncu_sass_wf.py <rep>"""
import csv, io, re, subprocess, sys, collections
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {k: hdr.index(k) for k in ('Source', 'Instructions Executed', 'L1 Wavefronts Shared', 'L1 Wavefronts Shared Ideal', '# Samples')}
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
tot = [0, 0, 0, 0]
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    src = r[ix['Source']].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', src).split(' ')[0]
    v = [float(r[ix[k]] or 0) for k in ('Instructions Executed', 'L1 Wavefronts Shared', 'L1 Wavefronts Shared Ideal', '# Samples')]
    for i in range(4):
        agg[op][i] += v[i]
        tot[i] += v[i]
print(f"{'opcode':18s} {'inst%':>7s} {'wf':>12s} {'wf/inst':>8s} {'ideal/inst':>10s} {'samples%':>8s}")
for op, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{op:18s} {100*v[0]/tot[0]:7.2f} {v[1]:12.0f} {v[1]/max(v[0],1):8.2f} {v[2]/max(v[0],1):10.2f} {100*v[3]/max(tot[3],1):8.2f}")
print('total inst', tot[0], 'wf', tot[1], 'ideal', tot[2])
