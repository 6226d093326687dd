import torch, statistics
n = 32 * 2**20
src = torch.empty(n, dtype=torch.uint8).pin_memory(); dst = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def one():
    dst.copy_(src, non_blocking=True)
def two():
    h = n // 2
    with torch.cuda.stream(s1): dst[:h].copy_(src[:h], non_blocking=True)
    with torch.cuda.stream(s2): dst[h:].copy_(src[h:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
def d2h():
    src.copy_(dst, non_blocking=True)
def both():
    with torch.cuda.stream(s1): dst.copy_(src, non_blocking=True)
    with torch.cuda.stream(s2): src2.copy_(dst2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
src2 = torch.empty(n, dtype=torch.uint8).pin_memory(); dst2 = torch.empty(n, dtype=torch.uint8, device='cuda')
for name, f in (('h2d 1 stream', one), ('h2d 2 streams', two), ('d2h', d2h), ('h2d+d2h concurrent', both)):
    ts = []
    for i in range(12):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts[2:]); print(name, round(ms, 3), 'ms', round(n / ms / 1e6, 1), 'GB/s')
