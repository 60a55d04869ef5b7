import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2409_14489_b200 import channel as ch
from paper_2409_14489_b200.config import LinkConfig
for lg in (8, 10, 12, 14, 17):
    n = 1 << lg
    lk = LinkConfig(num_spans=1, span_length_km=80.0, gamma_w_km=1.3)
    steps = ch.span_step_sizes(lk, ch.SimSettings(step_km=0.08), 1e-3)   # 1000 steps
    x = (torch.randn(1, 2, n, dtype=torch.complex128) * 1e-2).cuda()
    ch.propagate_tensor(x, lk, steps, 64e9)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ch.propagate_tensor(x, lk, steps, 64e9); b.record(); torch.cuda.synchronize()
    print(lg, f"{a.elapsed_time(b) / len(steps) * 1e3:.2f} us per fine step")
