import torch, time
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
