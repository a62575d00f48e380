"""Per-panel cycles of k_sep_inverse (RH_DEBUG=16): diag+loads, tile compute, barrier (CTA 0 and last)."""
import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gj_prof.bin", dtype=np.int64)
for name, o in (("cta0", 0), ("last", 512)):
    x = d[o:o + 512].reshape(-1, 4)
    x = x[x[:, 0] > 0]
    print(name, "panels", len(x), "diag+load %.0f  tile %.0f  barrier %.0f  (cycles, mean)" % (
        (x[:, 1] - x[:, 0]).mean(), (x[:, 2] - x[:, 1]).mean(), (x[:, 3] - x[:, 2]).mean()))
