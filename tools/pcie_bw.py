import torch, time
n = 1207959552 // 8
h_in = torch.empty(n, dtype=torch.int64).pin_memory(); h_out = torch.empty(n, dtype=torch.int64).pin_memory()
d_in = torch.empty(n, dtype=torch.int64, device="cuda"); d_out = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / k
def h2d(): d_in.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_out, non_blocking=True)
def both():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn); print(name, round(ms, 2), "ms", round(n * 8 / ms / 1e6, 1), "GB/s per direction")
