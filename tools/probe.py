"""FP64 pipe vs DMMA throughput on this GPU (tools/probe.py)."""
import ctypes, json, sys, torch
sys.path.insert(0, '.')
from paper_1806_07984_b200 import _lib
lib = _lib.load()
sink = torch.zeros(1, dtype=torch.float64, device='cuda')
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
out = {}
for name, fn, fl in (("dfma", lib.edg_probe_fp64, lambda b, it: b * 256 * 8 * it * 2),
                     ("dmma", lib.edg_probe_dmma, lambda b, it: b * 8 * 4 * it * 512)):
    best = 0
    for blocks in (nsm * 4, nsm * 8):
        for _ in range(3):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); _lib.check(fn(_lib.ptr(sink), blocks, 2048, st), name); b.record(); torch.cuda.synchronize()
            best = max(best, fl(blocks, 2048) / (a.elapsed_time(b) * 1e-3) / 1e12)
    out[name + "_tflops"] = best
print(json.dumps(out))
