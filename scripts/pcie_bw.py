import torch, time
n = 302 * 1024 * 1024 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
o = torch.empty(102 * 1024 * 1024 // 2, dtype=torch.bfloat16).pin_memory()
od = torch.empty_like(o, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f"H2D 302 MiB: {t:.3f} ms = {302*1.048576/t:.1f} GB/s")
e0.record()
for _ in range(10): o.copy_(od, non_blocking=True)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f"D2H 102 MiB: {t:.3f} ms = {102*1.048576/t:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(od, non_blocking=True)
torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"both directions concurrently: {e0.elapsed_time(e1)/10:.3f} ms per iteration")
