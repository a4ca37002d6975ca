# Context ceiling: cuBLAS DGEMM / ZGEMM throughput through torch.matmul (library, not the product).
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for dt, fl_per in ((torch.float64, 2), (torch.complex128, 8)):
    for n in (4096, 8192, 16384):
        a = torch.randn(n, n, dtype=dt, device="cuda"); b = torch.randn(n, n, dtype=dt, device="cuda")
        for _ in range(2): a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        reps = 5 if n < 16384 else 2
        e0.record()
        for _ in range(reps): a @ b
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{dt} n={n}: {fl_per*n**3/ms/1e9:.2f} TFLOP/s ({ms:.1f} ms)", flush=True)
        del a, b
# tall-skinny shapes like the filter: (N x N) @ (N x k)
for dt, fl_per in ((torch.float64, 2), (torch.complex128, 8)):
    for n, k in ((30000, 3000), (30000, 1000), (30000, 200)):
        a = torch.randn(n, n, dtype=dt, device="cuda"); b = torch.randn(n, k, dtype=dt, device="cuda")
        for _ in range(2): a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3): a @ b
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{dt} {n}x{n} @ {n}x{k}: {fl_per*n*n*k/ms/1e9:.2f} TFLOP/s ({ms:.1f} ms)", flush=True)
        del a, b
