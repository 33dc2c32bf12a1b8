import torch, time
n = 16 << 20
h1 = torch.empty(n, dtype=torch.float32).pin_memory(); h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d1 = torch.empty(n, dtype=torch.float32, device="cuda"); d2 = torch.empty(n, dtype=torch.float32, device="cuda")
S = [torch.cuda.Stream() for _ in range(8)]
def run(mode, splits):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10):
        for j in range(splits):
            sl = slice(j * n // splits, (j + 1) * n // splits)
            if mode in ("h2d", "both"):
                with torch.cuda.stream(S[j]): d1[sl].copy_(h1[sl], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(S[4 + j]): h2[sl].copy_(d2[sl], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(mode, splits, f"{10 * n * 4 / dt / 1e9:.1f} GB/s per direction, {dt / 10 * 1e3:.2f} ms per 64 MiB")
for mode in ["h2d", "d2h", "both"]:
    for sp in (1, 2, 4):
        run(mode, sp)
run("d2h", 1); run("both", 1)
