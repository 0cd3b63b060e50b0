"""Summarise lds_wf4 (3-D p=4 STP lane maps x flux storage orders): modelled
per-mapping wavefronts of the derivative loads and flux stores, as measured by
ncu.  python tools/probes/lds_wf4_report.py gpurun_out/ldswf4/out.csv"""
import collections
import csv
import sys

names = open(__file__.replace('_report.py', '_names.txt')).read().split()
rows = list(csv.reader(open(sys.argv[1])))
hdr, vals = None, {}
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        vals.setdefault(int(d['ID']), {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for i, n in enumerate(names):
    v = vals.get(i)
    if not v:
        continue
    if n.endswith('_st'):
        w = v['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum'] / max(v['smsp__inst_executed_op_shared_st.sum'], 1)
    else:
        w = v['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum'] / max(v['smsp__inst_executed_op_shared_ld.sum'], 1)
    parts = n.split('_')
    key = parts[0] + '_' + parts[1]
    kind = 'st' if n.endswith('_st') else parts[3]
    agg[key][kind].append(w)
for key, d in agg.items():
    s = '  '.join(f"{k}={sum(v) / len(v):.2f}" for k, v in sorted(d.items()))
    loads = sum(sum(d[a]) / len(d[a]) for a in ('a0', 'a1', 'a2'))
    print(f"{key:16s} {s}   loads/l-step={loads:.2f}")
