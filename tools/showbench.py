"""Summarise bench JSON lines: python tools/showbench.py <files...>"""
import json, sys
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith('{'):
            continue
        d = json.loads(line)
        ks = d.get('kernels', {})
        k = ks.get('stp_picard', {})
        c = ks.get('corrector_fused', {}) or ks.get('fv_patch', {})
        print(f"{f.split('/')[-1]:24s} value={d['value']:.3e} ms/step={d['ms_per_step']:.4f} stp_ms={k.get('ms_per_launch', 0):.4f} "
              f"frac={k.get('frac', 0):.3f} exec={k.get("executed_frac", 0):.3f} other_ms={c.get('ms_per_launch', 0):.4f} its={d['config'].get('picard_iterations_mean')}")
