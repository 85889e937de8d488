"""D2H bandwidth of one pinned copy against the same bytes split over several streams (tools only)."""
import torch, time
n = 1_258_494_894
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8).pin_memory()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
def one(): host.copy_(dev, non_blocking=True)
print("one copy      %.2f ms  %.1f GB/s" % (timed(one) * 1e3, n / timed(one) / 1e9))
for parts in (2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    step = (n + parts - 1) // parts
    def split():
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                host[i * step:(i + 1) * step].copy_(dev[i * step:(i + 1) * step], non_blocking=True)
    t = timed(split)
    print("%d streams     %.2f ms  %.1f GB/s" % (parts, t * 1e3, n / t / 1e9))
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
def h2d(): dev.copy_(h2, non_blocking=True)
t = timed(h2d); print("h2d one       %.2f ms  %.1f GB/s" % (t * 1e3, n / t / 1e9))
