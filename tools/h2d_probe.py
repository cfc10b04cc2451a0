import torch, time
dev = torch.device("cuda", 0)
h = torch.zeros(480, 640, dtype=torch.int16).pin_memory()
d = torch.empty_like(h, device=dev)
t = torch.zeros(3, 4, dtype=torch.float64).pin_memory()
td = torch.empty_like(t, device=dev)
s = torch.cuda.current_stream()
for name, fn in [("h2d depth", lambda: d.copy_(h, non_blocking=True)), ("h2d T", lambda: td.copy_(t, non_blocking=True)),
                 ("d2h T", lambda: t.copy_(td, non_blocking=True))]:
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(100): fn()
    e1.record(s); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 100 * 1e3, "us")
