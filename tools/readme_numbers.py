"""Regenerate the README / DESIGN measured tables from profiles/round1/bench*.json."""
import json
import re


def L(f):
    return json.loads(open('profiles/round1/' + f).read().strip().splitlines()[-1])


b, c1, c2, c3, c4, c5, r = (L(f) for f in ('bench.json', 'bench_cfg1.json', 'bench_cfg2_cfl02.json', 'bench_cfg3.json',
                                           'bench_cfg4.json', 'bench_cfg5.json', 'bench_reference.json'))


def stp(d):
    k = d['kernels']['stp_picard']
    return f"STP {100 * k['frac']:.1f} % of FP64 (executed {100 * k['executed_frac']:.1f} %)"


def cor(d):
    return f"corrector {100 * d['kernels']['corrector_fused']['frac']:.0f} % of HBM"


rows = [("cfg2 Euler 2-D p=5 243², CFL 0.9 (headline)", b, stp(b) + "; " + cor(b)),
        ("cfg2 at the parity-safe CFL 0.2", c2, stp(c2) + "; " + cor(c2)),
        ("cfg3 Euler 3-D p=4 64³", c3, stp(c3) + "; " + cor(c3)),
        ("cfg4 FV Euler 3-D 128³", c4, f"FV patch {100 * c4['kernels']['fv_patch']['frac']:.0f} % of HBM"),
        ("cfg5 AMR Euler 2-D p=3", c5, stp(c5) + "; " + cor(c5) + ", two streams"),
        ("cfg1 advection 2-D p=3 27²", c1, "launch-bound (729 cells)")]
out = ["| config | DoF-updates/s (device) | e2e (host buffers) | dominant kernel, fraction of its roofline |",
       "|---|---|---|---|"]
for n, d, s in rows:
    out.append(f"| {n} | {d['value']:.3g} | {d['e2e']['value']:.3g} | {s} |")
s = open('README.md').read()
i = s.index('| config | DoF-updates/s')
j = s.index('\n\n', i)
s = s[:i] + "\n".join(out) + s[j:]
s = re.sub(r"on \d+ host cores, cfg2\): [\d.e+]+ DoF-updates/s",
           f"on {r['cpu_baseline']['cores']} host cores, cfg2): {r['value']:.3g} DoF-updates/s", s)
open('README.md', 'w').write(s)


def krow(w, d, name):
    k = d['kernels'][name]
    ex = f" (executed {100 * k['executed_frac']:.1f} %)" if 'executed_frac' in k else ""
    return f"| {w} | {name} | {k['ms_per_launch']:.4f} | {k['achieved']:.1f} {k['unit']} | {100 * k['frac']:.1f} %{ex} |"


dr = ["| workload | kernel | ms per launch | achieved | fraction of roofline |", "|---|---|---|---|---|",
      krow('cfg2, CFL 0.9', b, 'stp_picard'), krow('cfg2, CFL 0.9', b, 'corrector_fused'),
      krow('cfg2, CFL 0.2', c2, 'stp_picard'), krow('cfg2, CFL 0.2', c2, 'corrector_fused'),
      krow('cfg3', c3, 'stp_picard'), krow('cfg3', c3, 'corrector_fused'),
      krow('cfg4', c4, 'fv_patch'),
      krow('cfg5', c5, 'stp_picard'), krow('cfg5', c5, 'corrector_fused')]
s = open('DESIGN.md').read()
i = s.index('| workload | kernel | ms per launch')
j = s.index('\n\n', i)
s = s[:i] + "\n".join(dr) + s[j:]
open('DESIGN.md', 'w').write(s)
print("\n".join(out))
print("\n".join(dr))
