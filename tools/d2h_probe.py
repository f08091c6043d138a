import torch, statistics
n = 66355200
dev = torch.empty(n, dtype=torch.uint8, device="cuda"); dev.fill_(3)
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for chunks in (1, 8, 32):
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step = n // chunks
        for c in range(chunks):
            host[c*step:(c+1)*step].copy_(dev[c*step:(c+1)*step], non_blocking=True)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"D2H pinned copy engine, {chunks} chunks: {statistics.median(ts):.3f} ms = {n/statistics.median(ts)/1e6:.1f} GB/s")
