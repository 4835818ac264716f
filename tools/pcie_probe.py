"""PCIe probe for the e2e leg: pinned H2D / D2H rates at the bench's transfer sizes, and
whether the two directions overlap."""
import torch

dev = torch.device("cuda", 0)
for mb in (4, 12, 40):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            if name == "h2d":
                d.copy_(h, non_blocking=True)
            elif name == "d2h":
                h.copy_(d, non_blocking=True)
            else:
                s1.wait_stream(torch.cuda.current_stream())
                s2.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
                torch.cuda.current_stream().wait_stream(s1)
                torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[name] = (ms, (2 if name == "both" else 1) * mb * (1 << 20) / (ms * 1e-3) / 1e9)
    print(f"{mb:3d} MB: " + "  ".join(f"{k} {v[0] * 1e3:7.1f} us {v[1]:6.1f} GB/s" for k, v in res.items()))
