import torch, time
x = torch.zeros(1, device='cuda')
N = 70
def work():
    for _ in range(N):
        x.add_(1)
for _ in range(10): work()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100): work()
e1.record(); torch.cuda.synchronize()
print("stream: us per kernel", e0.elapsed_time(e1) * 1000 / (100 * N))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    work()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        work()
torch.cuda.synchronize()
for _ in range(10): g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(100): g.replay()
e1.record(); torch.cuda.synchronize()
print("graph: us per kernel", e0.elapsed_time(e1) * 1000 / (100 * N))
