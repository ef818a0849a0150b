import torch, time
for mb in (2, 12, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device='cuda')
    for direction in ('h2d', 'd2h'):
        torch.cuda.synchronize()
        reps = 50
        t0 = time.perf_counter()
        for _ in range(reps):
            if direction == 'h2d': d.copy_(h, non_blocking=True)
            else: h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(mb, direction, round(n * reps / dt / 1e9, 1), 'GB/s')
