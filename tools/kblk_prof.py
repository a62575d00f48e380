"""Per-tile cycles of one k_blk MODE_U launch (RH_DEBUG=8): 8 warps' pieces, load wait, tops."""
import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kblk_prof.bin", dtype=np.int64).reshape(-1, 12)
d = d[d[:, 10] > 0]
pw = d[:, :8] & ((1 << 48) - 1)
nu = d[:, :8] >> 48
print("tiles", len(d))
print("pieces: max-warp mean %.0f, mean-warp mean %.0f cycles" % (pw.max(1).mean(), pw.mean()))
m = nu > 0
print("cycles per unit: mean %.0f (warps with units), max-warp units mean %.1f" % ((pw[m] / nu[m]).mean(), nu.max(1).mean()))
print("wait mean %.0f, tops mean %.0f, tile (ticket..pieces end) mean %.0f" % (d[:, 8].mean(), (d[:, 9] & ((1 << 48) - 1)).mean(), (d[:, 11] - d[:, 10]).mean()))

first = (d[:, 9] >> 48) & 1
tops = d[:, 9] & ((1 << 48) - 1)
for f in (1, 0):
    m = first == f
    if m.any():
        print("%s chunk of a ticket: tiles %d, wait mean %.0f, tops mean %.0f, pieces max-warp mean %.0f"
              % ("first" if f else "later", m.sum(), d[m, 8].mean(), tops[m].mean(), pw[m].max(1).mean()))
