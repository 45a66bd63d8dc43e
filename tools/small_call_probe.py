import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_05462_b200 as G
from paper_2408_05462_b200 import _abi
g = np.random.default_rng(4).normal(size=(6, 6, 6))
b = G.compress(g, 0.01)
G.decompress(b)
torch.cuda.synchronize()
import cProfile, pstats
t = time.perf_counter()
for _ in range(20): G.decompress(b)
print("decompress", (time.perf_counter() - t) / 20 * 1e3, "ms")
t = time.perf_counter()
for _ in range(20): G.compress(g, 0.01)
print("compress", (time.perf_counter() - t) / 20 * 1e3, "ms")
cProfile.run("for _ in range(10): G.decompress(b)", "/tmp/p.prof")
pstats.Stats("/tmp/p.prof").sort_stats("tottime").print_stats(10)
from paper_2408_05462_b200.blockcodec import CompressedBlock, HEADER_SIZE
from paper_2408_05462_b200 import exceptions as X
raw = bytearray(b.to_bytes())
times = []
for pos in range(HEADER_SIZE, min(len(raw), HEADER_SIZE + 40)):
    raw[pos] ^= 0x40
    t = time.perf_counter()
    try:
        G.decompress(CompressedBlock.from_bytes(bytes(raw)))
    except X.CorruptPayloadError:
        pass
    times.append((time.perf_counter() - t) * 1e3)
    raw[pos] ^= 0x40
print("corrupt decompress ms:", [round(x, 2) for x in times[:12]], "mean", sum(times) / len(times))
