import torch, time
torch.cuda.set_device(0)
n=537_000_000//4
h_in=torch.empty(n,dtype=torch.float32,pin_memory=True)
h_out=torch.empty(n,dtype=torch.float32,pin_memory=True)
d_a=torch.empty(n,dtype=torch.float32,device='cuda'); d_b=torch.empty(n,dtype=torch.float32,device='cuda')
s1,s2=torch.cuda.Stream(),torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a=time.perf_counter(); f(); torch.cuda.synchronize(); return (time.perf_counter()-a)*1e3
for _ in range(2):
    print("h2d", t(lambda: d_a.copy_(h_in, non_blocking=True)))
    print("d2h", t(lambda: h_out.copy_(d_b, non_blocking=True)))
    def both():
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    print("both", t(both))
