"""Host<->device copy bandwidth with pinned buffers (the e2e ceiling): H2D
alone, D2H alone, and both concurrently on two streams."""
import torch
dev = torch.device("cuda", 0)
n = 64 << 20  # 64 Mi halves = 128 MiB
h1 = torch.empty(n, dtype=torch.float16).pin_memory()
h2 = torch.empty(n, dtype=torch.float16).pin_memory()
d1 = torch.empty(n, dtype=torch.float16, device=dev)
d2 = torch.empty(n, dtype=torch.float16, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for st in (s1, s2): st.wait_event(a)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    for st in (s1, s2):
        e = torch.cuda.Event(); e.record(st); torch.cuda.current_stream().wait_event(e)
    b.record(); torch.cuda.synchronize()
    return reps * n * 2 / (a.elapsed_time(b) * 1e-3) / 1e9
for _ in range(2): run(True, True, 2)
print(f"H2D {run(True, False):.1f} GB/s, D2H {run(False, True):.1f} GB/s, "
      f"both concurrently {run(True, True):.1f} GB/s per direction")
