"""SURVEY.md 8(f) NEXT-3 ("measure before building it"): the direct-adjoint variant
replaces the transposed solves by H = Y_p + Z^T Y_x with Z = -J^-1 G_p for ALL
columns, i.e. one dense fp64 GEMM [n_p x n_x] x [n_x x n_p] (plus keeping Z,
n_x n_p 8 B).  Time that GEMM with cuBLAS (torch.matmul, fp64) at case9241's
shape and compare with the transposed-solve stages it would remove."""
import sys
import torch

n_x, n_p = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (17036, 2889)))
Z = torch.randn(n_x, n_p, dtype=torch.float64, device="cuda")
Y = torch.randn(n_x, n_p, dtype=torch.float64, device="cuda")
for _ in range(3):
    H = Z.t() @ Y
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    H = Z.t() @ Y
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
fl = 2.0 * n_p * n_p * n_x
print(f"Z^T Y_x GEMM {n_p}x{n_x}x{n_p} fp64: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s; Z holds {n_x * n_p * 8 / 1e6:.0f} MB")
