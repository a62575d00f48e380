import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kseg_timing.bin", dtype=np.int64).reshape(-1, 6)
t0 = d[:, 0].min()
st, sw, so = (d[:, 1] - d[:, 0]) / 1e3, (d[:, 2] - d[:, 1]) / 1e3, (d[:, 3] - d[:, 2]) / 1e3
print("CTAs", len(d), "span us %.1f" % ((d[:, 3].max() - t0) / 1e3), "super-levels per block: mean %.1f max %d" % (d[:, 5].mean(), d[:, 5].max()))
for nm, v in (("stage", st), ("sweep", sw), ("store", so), ("total", (d[:, 3] - d[:, 0]) / 1e3)):
    print(f"{nm:6s} mean {v.mean():7.2f} us  min {v.min():7.2f}  max {v.max():7.2f}")
sm = d[:, 4]
mid = t0 + (d[:, 3].max() - t0) / 2
print("CTAs per SM", np.bincount(sm).min(), np.bincount(sm).max(), "resident at mid", np.sum((d[:, 0] <= mid) & (d[:, 3] >= mid)))
