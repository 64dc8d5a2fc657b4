"""Host -> device copy bandwidth from pinned memory: one stream vs two concurrent streams (TOOL)."""
import torch

n = 512 << 20  # bytes
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    one = n / (e0.elapsed_time(e1) / 1e3) / 1e9
    h = n // 2
    torch.cuda.synchronize()
    e0.record()
    s1.wait_event(e0); s2.wait_event(e0)
    with torch.cuda.stream(s1):
        dst[:h].copy_(src[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dst[h:].copy_(src[h:], non_blocking=True)
    ev1, ev2 = torch.cuda.Event(), torch.cuda.Event()
    ev1.record(s1); ev2.record(s2)
    torch.cuda.current_stream().wait_event(ev1); torch.cuda.current_stream().wait_event(ev2)
    e1.record()
    torch.cuda.synchronize()
    two = n / (e0.elapsed_time(e1) / 1e3) / 1e9
    print({"one_stream_GBs": round(one, 1), "two_streams_GBs": round(two, 1)})
