"""Host->device bandwidth from pinned memory: one copy vs chunked copies on
several streams (what the e2e leg's upload of A can reach)."""
import time

import torch

nbytes = 4 << 30
h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty_like(h, device="cuda")
for nst in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    chunks = h.chunk(nst * 4)
    dchunks = d.chunk(nst * 4)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, (a, b) in enumerate(zip(chunks, dchunks)):
            with torch.cuda.stream(streams[i % nst]):
                b.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{nst} streams: {nbytes / dt / 1e9:.1f} GB/s")
t0 = time.perf_counter()
x = h[: (1 << 30) // 8].numpy()
y = torch.from_numpy(x).to("cuda")
torch.cuda.synchronize()
print(f"from_numpy(pinned view).to(cuda) 1 GiB: {(1 << 30) / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
