import torch
for ns, N in ((521, 1024), (2240, 1024)):
    A = torch.randn(ns, ns, dtype=torch.float64, device="cuda")
    B = torch.randn(ns, N, dtype=torch.float64, device="cuda")
    C = torch.empty(ns, N, dtype=torch.float64, device="cuda")
    for _ in range(5): torch.matmul(A, B, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): torch.matmul(A, B, out=C)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(ns, N, "cuBLAS dgemm %.1f us, %.1f TF" % (ms * 1e3, 2 * ns * ns * N / ms / 1e9))
