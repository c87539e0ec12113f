"""Host->device bandwidth of a 1 GiB pinned buffer: one cudaMemcpyAsync vs the same bytes split
over 2 / 4 streams (copy engines), and chunked on one stream."""
import torch

n = 1 << 28
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
h.fill_(1.0)


def run(parts, streams):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_event(e0)
    step = n // parts
    for i in range(parts):
        with torch.cuda.stream(ss[i % streams]):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    for s in ss:
        e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return 4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9


for parts, streams in [(1, 1), (2, 2), (4, 4), (8, 2), (16, 1), (64, 4)]:
    bw = sorted(run(parts, streams) for _ in range(5))[2]
    print(f"H2D 1 GiB: {parts} chunks over {streams} streams: {bw:.1f} GB/s")
