"""Pinned host->device copy bandwidth on the box (1 stream, 2 streams, 64 pieces): the e2e
critical path streams the LOD-20/60 levels at this rate (measured r2: ~55 GB/s in every form)."""
import torch, time
n = 1600 * 1024 * 1024
a = torch.empty(n, dtype=torch.uint8).pin_memory(); b = torch.empty(n, dtype=torch.uint8).pin_memory()
da = torch.empty(n, dtype=torch.uint8, device='cuda'); db = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    # many small pieces
    with torch.cuda.stream(s1):
        for k in range(64): da[k*(n//64):(k+1)*(n//64)].copy_(a[k*(n//64):(k+1)*(n//64)], non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"1 stream {n/(t1-t)/1e9:.1f} GB/s; 2 streams {2*n/(t2-t1)/1e9:.1f} GB/s; 64 pieces {n/(t3-t2)/1e9:.1f} GB/s")
