import os
import time

import torch
n = 514*514*514
X=514; pitch=528
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(514*514*pitch, dtype=torch.float64, device='cuda')
s = torch.cuda.current_stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter()-t0)/reps
import ctypes
cudart = ctypes.CDLL('libcudart.so') if False else None
dflat = d[:n]
print("H2D contiguous GB/s", n*8/t(lambda: dflat.copy_(h, non_blocking=True))/1e9)
print("D2H contiguous GB/s", n*8/t(lambda: h.copy_(dflat, non_blocking=True))/1e9)
d2 = d.view(514*514, pitch)[:, :X]
h2 = h.view(514*514, X)
print("H2D 2D pitched GB/s", n*8/t(lambda: d2.copy_(h2, non_blocking=True))/1e9)
print("D2H 2D pitched GB/s", n*8/t(lambda: h2.copy_(d2, non_blocking=True))/1e9)

# device-to-device pitched copy through the copy engine (cudaMemcpy2DAsync), as the staged upload uses
import ctypes
rt = ctypes.CDLL("libcudart.so.12")
dsrc = torch.empty(n, dtype=torch.float64, device="cuda")
def d2d2():
    rc = rt.cudaMemcpy2DAsync(ctypes.c_void_p(d.data_ptr()), ctypes.c_size_t(pitch * 8),
                              ctypes.c_void_p(dsrc.data_ptr()), ctypes.c_size_t(X * 8), ctypes.c_size_t(X * 8),
                              ctypes.c_size_t(514 * 514), ctypes.c_int(3), ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, rc
print("D2D 2D pitched (copy engine) GB/s (read+write)", 2 * n * 8 / t(d2d2) / 1e9)

# concurrency: two H2D streams at once, H2D with a concurrent D2H, and 67 MB chunks (the staged upload's)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2


def h2d_two_streams():
    with torch.cuda.stream(s1):
        dflat[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        dflat[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.synchronize()


print("H2D two streams GB/s", n * 8 / t(h2d_two_streams) / 1e9)
hout = torch.empty(n // 8, dtype=torch.float64).pin_memory()
dout = torch.empty(n // 8, dtype=torch.float64, device="cuda")


def h2d_with_d2h():
    with torch.cuda.stream(s1):
        dflat.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    torch.cuda.synchronize()


print("H2D (8 B/cell) with a concurrent D2H of 1/8 the bytes: H2D-equivalent GB/s", n * 8 / t(h2d_with_d2h) / 1e9)
chunk = 32 * 514 * 514


def h2d_chunks():
    for z in range(0, n, chunk):
        e = min(n, z + chunk)
        dflat[z:e].copy_(h[z:e], non_blocking=True)


print("H2D in 67 MB chunks GB/s", n * 8 / t(h2d_chunks) / 1e9)
