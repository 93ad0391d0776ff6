import torch, time
dev = torch.device("cuda", 0)
n = 4 << 30  # 4 GiB
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
th = t(h2d); td = t(d2h); tb = t(both)
print(f"H2D {n/th/1e9:.1f} GB/s  D2H {n/td/1e9:.1f} GB/s  both: {2*n/tb/1e9:.1f} GB/s total ({n/tb/1e9:.1f} per direction)")
