"""Per-block phase cycles of k_fact_blocks (RH_DEBUG=128): staging, pieces, tops T1, tops T2."""
import numpy as np, sys
d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fact_prof.bin", dtype=np.int64).reshape(-1, 8)
st, pc, t1, t2 = d[:, 1] - d[:, 0], d[:, 2] - d[:, 1], d[:, 3] - d[:, 2], d[:, 4] - d[:, 3]
for nm, v in (("stage", st), ("pieces", pc), ("tops T1", t1), ("tops T2", t2), ("total", d[:, 4] - d[:, 0])):
    print(f"{nm:8s} mean {v.mean():8.0f}  max {v.max():8.0f} cycles")
