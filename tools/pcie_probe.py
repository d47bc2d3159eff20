"""Pinned host<->device copy bandwidth on this box: h2d alone, d2h alone, both at once
(separate streams), for the C2 end-to-end sizes (22.15 MB in, 33.2 MB out)."""
import torch

dev = torch.device("cuda", 0)
nin, nout = 22151168 // 4, 33226752 // 4
hin = torch.empty(nin, pin_memory=True); hout = torch.empty(nout, pin_memory=True)
din = torch.empty(nin, device=dev); dout = torch.empty(nout, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


t_in = timed(lambda: din.copy_(hin, non_blocking=True))
t_out = timed(lambda: hout.copy_(dout, non_blocking=True))
t_both = timed(both)
print(f"h2d {t_in*1e3:.0f} us ({nin*4/t_in/1e6:.1f} GB/s)  d2h {t_out*1e3:.0f} us ({nout*4/t_out/1e6:.1f} GB/s)  "
      f"both {t_both*1e3:.0f} us (sum {(t_in+t_out)*1e3:.0f})")
