"""cuBLAS DGEMM (torch) at the separator product's shape: [ns x ns] x [ns x N] fp64."""
import sys
import torch
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 521
for N in (963, 1024, 362):
    A = torch.randn(ns, ns, dtype=torch.float64, device="cuda")
    B = torch.randn(ns, N, dtype=torch.float64, device="cuda")
    C = torch.empty(ns, N, dtype=torch.float64, device="cuda")
    for _ in range(5):
        torch.matmul(A, B, out=C)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(50):
        torch.matmul(A, B, out=C)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 50 * 1e-3
    print(f"ns={ns} N={N}: {t*1e6:.1f} us, {2*ns*ns*N/t/1e12:.1f} TFLOP/s")
