"""PCIe bandwidth of chr_sm_copy (UVA copy kernel) vs the DMA engines, H2D /
D2H alone and concurrently, for several CTA counts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_05462_b200 import _abi  # noqa: E402

L = _abi.lib()
torch.cuda.set_device(0)
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best * 1e3


def sm(dst, src, ctas, st):
    L.chr_sm_copy(dst.data_ptr(), src.data_ptr(), n, ctas, st.cuda_stream)


print("dma h2d %.2f ms  d2h %.2f ms" % (t(lambda: d_a.copy_(h_in, non_blocking=True)),
                                        t(lambda: h_out.copy_(d_b, non_blocking=True))))


def dma_both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


print("dma both %.2f ms" % t(dma_both))
for ctas in (8, 16, 32, 64, 128, 148, 296):
    a = t(lambda: sm(d_a, h_in, ctas, s1))
    b = t(lambda: sm(h_out, d_b, ctas, s1))

    def both():
        sm(d_a, h_in, ctas, s1)
        sm(h_out, d_b, ctas, s2)
    c = t(both)
    print(f"sm ctas={ctas:4d}: h2d {a:.2f} ms ({n / a / 1e6:.1f} GB/s)  d2h {b:.2f} ms ({n / b / 1e6:.1f} GB/s)  "
          f"both {c:.2f} ms")
