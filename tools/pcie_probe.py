"""PCIe strategies for the e2e step: one contiguous vs five tensors, chunked bidirectional copies."""
import time
import torch
dev = torch.device("cuda")
n = 24_000_000 // 4
hin = torch.empty(n, dtype=torch.float32).pin_memory()
hout = torch.empty(n, dtype=torch.float32).pin_memory()
din = torch.empty(n, dtype=torch.float32, device=dev)
dout = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, k=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3
def both(chunks):
    c = n // chunks
    for i in range(chunks):
        with torch.cuda.stream(s1):
            din[i*c:(i+1)*c].copy_(hin[i*c:(i+1)*c], non_blocking=True)
        with torch.cuda.stream(s2):
            hout[i*c:(i+1)*c].copy_(dout[i*c:(i+1)*c], non_blocking=True)
print(f"H2D contiguous {timed(lambda: din.copy_(hin, non_blocking=True)):.3f} ms, D2H {timed(lambda: hout.copy_(dout, non_blocking=True)):.3f} ms")
for ch in (1, 2, 4, 8, 24):
    print(f"both directions, {ch} chunks: {timed(lambda: both(ch)):.3f} ms")
