import time, torch
t = torch.empty((1700, 2400, 3), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
keep = None
for it in range(6):
    t0 = time.perf_counter()
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    t1 = time.perf_counter()
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    a = h.numpy()
    keep = a
    print(f"alloc {(t1-t0)*1e3:.2f} ms copy {(t2-t1)*1e3:.2f} ms")
# reuse one pinned buffer
h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
for it in range(3):
    t1 = time.perf_counter(); h.copy_(t, non_blocking=True); torch.cuda.current_stream().synchronize(); t2 = time.perf_counter()
    print(f"reuse copy {(t2-t1)*1e3:.2f} ms")
