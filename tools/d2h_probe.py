"""PCIe probe for the streaming e2e: one 378 MB pinned D2H on one stream vs
split across 2 / 4 streams, and the latency of a small synchronous D2H
(the session's control-block read) while a large copy is in flight."""
import time

import torch

dev = torch.device("cuda:0")
n = 378 * 2**20 // 4
src = torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device=dev)
dst = torch.empty(n, dtype=torch.int32).pin_memory()
streams = [torch.cuda.Stream() for _ in range(4)]


def copy(parts):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = (n + parts - 1) // parts
    for i in range(parts):
        with torch.cuda.stream(streams[i]):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for parts in (1, 2, 4, 1, 2, 4):
    t = copy(parts)
    print(f"D2H 378 MB over {parts} stream(s): {t*1e3:.2f} ms  {n*4/t/1e9:.1f} GB/s")
small = torch.zeros(16, dtype=torch.int64, device=dev)
for trial in range(3):
    torch.cuda.synchronize()
    with torch.cuda.stream(streams[0]):
        dst.copy_(src, non_blocking=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(streams[1]):
        v = small.cpu()  # synchronous small D2H on another stream
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"small D2H during big copy: {(t1-t0)*1e3:.3f} ms (big copy done after {(t2-t0)*1e3:.2f} ms)")
