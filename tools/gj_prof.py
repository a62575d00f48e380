"""Per-panel cycles of k_sep_inverse (RH_DEBUG=16): CTA 0 (diag+loads, tile compute,
barrier) and the lookahead CTA (its work, barrier)."""
import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gj_prof.bin", dtype=np.int64)
x = d[0:512].reshape(-1, 4)
x = x[x[:, 0] > 0]
print("cta0", "panels", len(x), "diag+load %.0f  tile %.0f  barrier %.0f  (cycles, mean)" % (
    (x[:, 1] - x[:, 0]).mean(), (x[:, 2] - x[:, 1]).mean(), (x[:, 3] - x[:, 2]).mean()))
y = d[512:1024].reshape(-1, 4)
y = y[y[:, 0] > 0]
print("helper", "panels", len(y), "work %.0f  barrier %.0f  (cycles, mean)" % (
    (y[:, 2] - y[:, 0]).mean(), (y[:, 3] - y[:, 2]).mean()))
z = y[y[:, 1] > y[:, 0]]
print("helper split: loads+update %.0f  invert+publish %.0f" % ((z[:, 1] - z[:, 0]).mean(), (z[:, 2] - z[:, 1]).mean()))
