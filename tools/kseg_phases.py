"""Per-CTA phase cycles of one k_seg launch (RH_DEBUG=8 dump, see redhess.cu)."""
import numpy as np
import sys

d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kseg_phases.bin", dtype=np.int64).reshape(-1, 20)
pw = d[:, :16]
print("CTAs", len(d))
print("piece cycles: max-over-warps mean %.0f max %d; mean-over-warps %.0f" % (pw.max(1).mean(), pw.max(), pw.mean()))
print("tops gather cycles mean %.0f max %d; dense+store mean %.0f max %d; tops mean %.1f" %
      (d[:, 16].mean(), d[:, 16].max(), d[:, 17].mean(), d[:, 17].max(), d[:, 18].mean()))
i = int(np.argmax(pw.max(1)))
print("worst CTA", i, "warps:", pw[i].tolist())
