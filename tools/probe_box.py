"""Probe the GPU box: device props, host cores, pinned H2D/D2H bandwidth."""
import os, time, json, subprocess
import torch
out = {}
out["cpu_count"] = os.cpu_count()
try:
    import psutil
    out["physical_cores"] = psutil.cpu_count(logical=False)
except Exception as e:
    out["physical_cores"] = str(e)
p = torch.cuda.get_device_properties(0)
out["gpu"] = p.name; out["sms"] = p.multi_processor_count; out["mem_gb"] = p.total_memory / 1e9
out["l2"] = getattr(p, "L2_cache_size", None)
for mb in (16, 128, 512):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); [d.copy_(h, non_blocking=True) for _ in range(5)]; e.record(); e.synchronize()
    out[f"h2d_{mb}MB_GBs"] = 5 * n / (s.elapsed_time(e) * 1e-3) / 1e9
    s.record(); [h.copy_(d, non_blocking=True) for _ in range(5)]; e.record(); e.synchronize()
    out[f"d2h_{mb}MB_GBs"] = 5 * n / (s.elapsed_time(e) * 1e-3) / 1e9
    # bidirectional
    s2 = torch.cuda.Stream()
    d2 = torch.empty_like(d); h2 = torch.empty_like(h).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    out[f"bidir_{mb}MB_GBs_each"] = 5 * n / (time.perf_counter() - t0) / 1e9
print(json.dumps(out, indent=1))
