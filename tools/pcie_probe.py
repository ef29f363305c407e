import torch, time
n = 31457280 // 8
h = torch.empty(n, dtype=torch.int64).pin_memory(); d = torch.empty(n, dtype=torch.int64, device='cuda')
h2 = torch.empty(n, dtype=torch.int64).pin_memory(); d2 = torch.empty(n, dtype=torch.int64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ('h2d', 'd2h', 'both'):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20):
        if mode in ('h2d', 'both'):
            with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        if mode in ('d2h', 'both'):
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(mode, round(20 * n * 8 / dt / 1e9, 1), 'GB/s per direction')
