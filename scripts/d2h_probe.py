"""PCIe read-back rate on the GPU box: one D2H copy vs two / four concurrent copies (streams)."""
import torch, time
n = 1 << 30
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{k} stream(s): {n / dt / 1e9:.1f} GB/s")
h = torch.empty(n // 4, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter(); src[: n // 4].copy_(h, non_blocking=True); torch.cuda.synchronize()
print(f"H2D: {n / 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
