"""Host link on this box at the e2e leg's transfer size (one configs[4] c128
waveform = 268 MB): H2D alone, D2H alone, both at once (GB/s each)."""
import torch
n = 268435456
hx = torch.empty(n, dtype=torch.uint8).pin_memory()
ho = torch.empty(n, dtype=torch.uint8).pin_memory()
dx = torch.empty(n, dtype=torch.uint8, device="cuda")
do = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
R = 20


def timed(h2d, d2h):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    if h2d:
        with torch.cuda.stream(s1):
            ev[0].record()
            for _ in range(R):
                dx.copy_(hx, non_blocking=True)
            ev[1].record()
    if d2h:
        with torch.cuda.stream(s2):
            ev[2].record()
            for _ in range(R):
                ho.copy_(do, non_blocking=True)
            ev[3].record()
    torch.cuda.synchronize()
    out = []
    if h2d:
        out.append(f"h2d {n * R / ev[0].elapsed_time(ev[1]) / 1e6:.1f} GB/s")
    if d2h:
        out.append(f"d2h {n * R / ev[2].elapsed_time(ev[3]) / 1e6:.1f} GB/s")
    return ", ".join(out)


for _ in range(2):
    print("alone:", timed(True, False), "|", timed(False, True))
    print("concurrent:", timed(True, True))
