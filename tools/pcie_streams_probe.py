"""D2H / H2D bandwidth of pinned copies with 1, 2 and 4 concurrent streams
(is one copy stream enough to saturate PCIe for the y drain?)."""
import torch

N = 64 * 2**20
dev = torch.device("cuda:0")
src = torch.empty(N, dtype=torch.uint8, device=dev)
dst = torch.empty(N, dtype=torch.uint8).pin_memory()
hsrc = torch.empty(N, dtype=torch.uint8).pin_memory()
for direction in ("d2h", "h2d"):
    for k in (1, 2, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(k)]
        part = N // k
        best = 1e9
        for rep in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i, s in enumerate(streams):
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    if direction == "d2h":
                        dst[i * part:(i + 1) * part].copy_(src[i * part:(i + 1) * part], non_blocking=True)
                    else:
                        src[i * part:(i + 1) * part].copy_(hsrc[i * part:(i + 1) * part], non_blocking=True)
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{direction} streams={k}: {N / best / 1e6:.1f} GB/s")
