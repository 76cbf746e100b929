"""H2D copy rate: one 24.5 MB copy vs three 8.2 MB copies, int16 pinned."""
import torch

dev = torch.device("cuda", 0)
big_h = torch.empty((3 * 1700, 2400), dtype=torch.int16).pin_memory()
big_d = torch.empty(big_h.shape, dtype=torch.int16, device=dev)
parts_h = [torch.empty((1700, 2400), dtype=torch.int16).pin_memory() for _ in range(3)]
parts_d = [torch.empty((1700, 2400), dtype=torch.int16, device=dev) for _ in range(3)]
f32_h = torch.empty((1700, 2400, 3), dtype=torch.float32).pin_memory()
f32_d = torch.empty(f32_h.shape, dtype=torch.float32, device=dev)


def rate(fn, nbytes, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * n / (e0.elapsed_time(e1) / 1e3) / 1e9


print("H2D one 24.5 MB int16: %.1f GB/s" % rate(lambda: big_d.copy_(big_h, non_blocking=True), big_h.numel() * 2))
print("H2D 3 x 8.2 MB int16: %.1f GB/s" % rate(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(parts_d, parts_h)], 3 * parts_h[0].numel() * 2))
print("H2D 49 MB float32: %.1f GB/s" % rate(lambda: f32_d.copy_(f32_h, non_blocking=True), f32_h.numel() * 4))
print("D2H 49 MB float32: %.1f GB/s" % rate(lambda: f32_h.copy_(f32_d, non_blocking=True), f32_h.numel() * 4))
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
