"""H2D throughput while a D2H stream is busy: one copy vs pieces."""
import time, torch
n = 125 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
h_out = torch.empty(4 * n, dtype=torch.uint8).pin_memory()
d_out = torch.empty(4 * n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d(pieces):
    step = n // pieces
    with torch.cuda.stream(s1):
        for i in range(pieces):
            d_in[i*step:(i+1)*step].copy_(h_in[i*step:(i+1)*step], non_blocking=True)
for pieces in (1, 14):
    for bidir in (False, True):
        torch.cuda.synchronize()
        if bidir:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)  # ~9 ms of D2H
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1); h2d(pieces); e1.record(s1); e1.synchronize()
        torch.cuda.synchronize()
        print(f"pieces={pieces:2d} bidir={bidir}: H2D {n/ (e0.elapsed_time(e1)*1e-3)/1e9:.1f} GB/s")
