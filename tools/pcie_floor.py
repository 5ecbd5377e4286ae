import torch, time
n_h2d = 412350144 // 8; n_d2h = 137624768 // 8
h = torch.empty(n_h2d, dtype=torch.float64).pin_memory(); d = torch.empty(n_h2d, dtype=torch.float64, device='cuda')
h2 = torch.empty(n_d2h, dtype=torch.float64).pin_memory(); d2 = torch.empty(n_d2h, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
    print(f"h2d {n_h2d*8/t1/1e9:.1f} GB/s ({t1*1e3:.2f} ms), d2h {n_d2h*8/t2/1e9:.1f} GB/s ({t2*1e3:.2f} ms), both {t3*1e3:.2f} ms")
