"""Summarise bench JSON lines: python tools/summ.py gpurun_out/<tag>/bench_*.json"""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    k = d.get("kernels", {})
    ks = " ".join(f"{n}:{v['ms_per_launch']:.3f}ms/{(v['frac'] or 0)*100:.1f}%" for n, v in k.items())
    var = d.get("parity_safe_variant") or {}
    print(f"{f.split('/')[-1]:24s} value={d['value']:.3e} ms/step={d['ms_per_step']:.3f} its={d['config'].get('picard_iterations_mean')} "
          f"roof={((d['roofline']['frac'] or 0)*100):.1f}% {ks} e2e={(d.get('e2e') or {}).get('value', 0):.3e} "
          f"var={var.get('value', 0):.3e}/{(var.get('roofline_frac') or 0)*100:.1f}% nonfinite={d['config'].get('nonfinite_cell_results')} first={d['config'].get('first_nonfinite_step')}")
