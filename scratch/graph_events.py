import torch, time
x = torch.randn(1 << 24, device='cuda'); y = torch.empty_like(x)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    y.copy_(x)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    e[0].record()
    y.copy_(x)
    e[1].record()
    y.mul_(2.0)
    e[2].record()
for _ in range(5): g.replay()
torch.cuda.synchronize()
try:
    print("in-graph elapsed:", e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]))
except Exception as ex:
    print("in-graph elapsed failed:", ex)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(100): g.replay()
t1.record(); torch.cuda.synchronize()
print("per replay", t0.elapsed_time(t1) / 100)
