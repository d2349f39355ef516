import torch, time
n = 512 << 20
h = torch.empty(n, dtype=torch.int8).pin_memory()
d = torch.empty(n, dtype=torch.int8, device="cuda")
for chunks in (1, 4, 16, 64):
    torch.cuda.synchronize()
    s = [torch.cuda.Stream() for _ in range(2)]
    t0 = time.perf_counter()
    for it in range(5):
        c = n // chunks
        for i in range(chunks):
            with torch.cuda.stream(s[i % 2]):
                d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"chunks {chunks}: {n/dt/1e9:.1f} GB/s")
