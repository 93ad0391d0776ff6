"""PCIe copy rates between pinned host memory and the device: H2D alone, D2H alone, both
directions at once, in one copy or split into chunks over several streams.

  python tools/pcie_bw.py [GiB]
"""
import sys
import time

import torch

dev = torch.device("cuda", 0)
n = int(float(sys.argv[1]) * (1 << 30)) if len(sys.argv) > 1 else 4 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream() for _ in range(8)]


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps


def copy(dst, src, nstreams, base):
    ch = (n + nstreams - 1) // nstreams
    for i in range(nstreams):
        with torch.cuda.stream(streams[base + i]):
            dst[i * ch:(i + 1) * ch].copy_(src[i * ch:(i + 1) * ch], non_blocking=True)


for ns in (1, 2, 4):
    th = t(lambda: copy(d1, h1, ns, 0))
    td = t(lambda: copy(h2, d2, ns, 4))
    tb = t(lambda: (copy(d1, h1, ns, 0), copy(h2, d2, ns, 4)))
    print(f"{n / 2**30:.0f} GiB, {ns} stream(s) per direction: H2D {n / th / 1e9:.1f} GB/s  D2H {n / td / 1e9:.1f} GB/s  "
          f"both: {2 * n / tb / 1e9:.1f} GB/s total ({n / tb / 1e9:.1f} per direction)", flush=True)
