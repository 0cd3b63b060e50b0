"""Per-instruction shared-memory wavefronts (top N by wavefronts): python tools/ncu_sass_lds.py <rep> [N]"""
import csv, io, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
I = lambda k: hdr.index(k)
recs = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    ex = float(r[I('Instructions Executed')] or 0)
    wf = float(r[I('L1 Wavefronts Shared')] or 0)
    idl = float(r[I('L1 Wavefronts Shared Ideal')] or 0)
    if wf > 0:
        recs.append((wf, ex, idl, r[I('Address')][-5:], r[I('Source')].strip()[:70]))
recs.sort(reverse=True)
for wf, ex, idl, a, s in recs[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{a} {s:70s} ex={ex:10.0f} wf/inst={wf/ex:5.2f} ideal={idl/ex:5.2f}")
