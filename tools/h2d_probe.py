"""Pinned H2D bandwidth of a 400 MB list: one stream vs chunks over two streams (dev tool)."""
import torch
n = 100_000_000
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for nst, nch in ((1, 1), (1, 11), (2, 12), (2, 24), (3, 24), (4, 24)):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    per = (n + nch - 1) // nch
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in streams:
            st.wait_stream(torch.cuda.current_stream())
        for c in range(nch):
            st = streams[c % nst]
            with torch.cuda.stream(st):
                d[c * per:(c + 1) * per].copy_(h[c * per:(c + 1) * per], non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"streams={nst} chunks={nch}: {best:.3f} ms = {n * 4 / best / 1e6:.1f} GB/s")
