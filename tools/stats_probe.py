import sys, torch, time
sys.path.insert(0, '.')
from paper_2408_05462_b200 import device as D
torch.cuda.set_device(0)
n = int(sys.argv[1]); m = int(sys.argv[2])
vol = torch.rand(n * n * n, device='cuda', dtype=torch.float32)
cands = [float(x) for x in torch.linspace(0.05, 0.95, m)]
for _ in range(3):
    D.stats(vol, (n, n, n), 32, cands)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    D.stats(vol, (n, n, n), 32, cands)
b.record(); torch.cuda.synchronize()
print(n, m, a.elapsed_time(b) / 5, "ms", 4 * n**3 / (a.elapsed_time(b) / 5 * 1e-3) / 1e9, "GB/s")
