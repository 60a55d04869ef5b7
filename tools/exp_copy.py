import torch, time
x = torch.empty((1, 2, 1 << 20), dtype=torch.complex64).pin_memory()
d = torch.empty_like(x, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): fn()
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 50
    print(name, f"{t:.3f} ms", f"{x.numel()*8/t/1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x2 = torch.empty_like(x).pin_memory(); d2 = torch.empty_like(d)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    with torch.cuda.stream(s1): d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): x2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
b.record(); torch.cuda.synchronize()
print("h2d+d2h concurrent", f"{a.elapsed_time(b)/50:.3f} ms")
