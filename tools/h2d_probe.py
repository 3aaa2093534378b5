import torch, time
n = 490
src = [torch.empty((54, 131072), dtype=torch.int32).pin_memory() for _ in range(n)]
dst = torch.empty((n, 54, 131072), dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        for i in range(n):
            with torch.cuda.stream(ss[i % streams]):
                dst[i].copy_(src[i], non_blocking=True)
        torch.cuda.synchronize(); dt = time.time() - t
    print(streams, "streams:", round(n * 54 * 131072 * 4 / dt / 1e9, 1), "GB/s", round(dt * 1e3, 1), "ms")
