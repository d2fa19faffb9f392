import torch, time
for mb in (5.2, 537):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    a, b, c = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    a.record(); d.copy_(h, non_blocking=True); b.record(); h.copy_(d, non_blocking=True); c.record()
    torch.cuda.synchronize()
    print(f"{mb} MB: H2D {a.elapsed_time(b)*1e3:.1f} us ({mb*1e6/a.elapsed_time(b)/1e6:.1f} GB/s), D2H {b.elapsed_time(c)*1e3:.1f} us ({mb*1e6/b.elapsed_time(c)/1e6:.1f} GB/s)")
