import torch, time
dev = torch.device("cuda", 0)
for nbytes in (393216, 524288, 1 << 20, 4 << 20):
    h = torch.empty(nbytes // 2, dtype=torch.bfloat16).pin_memory()
    d = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev)
    for direction in ("h2d", "d2h"):
        evs = []
        for i in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            a.record()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in evs[5:])
        print(direction, nbytes, "median us", round(t[len(t)//2] * 1e3, 1), "GB/s", round(nbytes / (t[len(t)//2] * 1e-3) / 1e9, 1))
