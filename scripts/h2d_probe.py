import torch, time
n = 600_000_000
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
h.fill_(7)
d = torch.empty(n, dtype=torch.int64, device="cuda")
for chunk in (1 << 25, 1 << 27, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for b in range(0, n, chunk):
        d[b:b + chunk].copy_(h[b:b + chunk], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print("chunk", chunk, "GB/s", round(n * 8 / ms / 1e6, 1))
# two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
half = n // 2
with torch.cuda.stream(s1):
    d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2):
    d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize()
print("2 streams GB/s", round(n * 8 / (time.perf_counter() - t) / 1e9, 1))

# full duplex: 4 MB H2D and 8 MB D2H concurrently on two streams vs back to back
hk = torch.empty(1_000_000, dtype=torch.int32, pin_memory=True)
hy = torch.empty(1_000_000, dtype=torch.float64, pin_memory=True)
dk = torch.empty(1_000_000, dtype=torch.int32, device="cuda")
dy = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    xs = []
    for _ in range(reps + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        xs.append((time.perf_counter() - t0) * 1e6)
    return round(sorted(xs[3:])[reps // 2], 1)


def seq():
    dk.copy_(hk, non_blocking=True)
    hy.copy_(dy, non_blocking=True)


def duplex():
    with torch.cuda.stream(up):
        dk.copy_(hk, non_blocking=True)
    with torch.cuda.stream(down):
        hy.copy_(dy, non_blocking=True)


print("4MB H2D + 8MB D2H back to back us", timed(seq), " concurrent us", timed(duplex))
