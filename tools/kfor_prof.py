"""Per-CTA phase cycles of one k_for launch (RH_DEBUG=8192): barrier arm, row-copy issue, fill, copy wait, compute."""
import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kfor_prof.bin", dtype=np.int64).reshape(-1, 6)
d = d[d[:, 0] > 0]
print("CTAs", len(d))
for name, a, b in (("arm", 0, 1), ("row copies", 1, 2), ("fill", 2, 3), ("copy wait", 3, 4), ("compute+store", 4, 5), ("total", 0, 5)):
    v = d[:, b] - d[:, a]
    print("%-14s mean %7.0f  p50 %7.0f  p90 %7.0f cycles" % (name, v.mean(), np.median(v), np.percentile(v, 90)))
