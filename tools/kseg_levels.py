import numpy as np, sys
sys.path.insert(0, '.')
import gridgen, paper_2201_00241_b200 as rh
d = np.fromfile("gpurun_out/kseg_levels.bin", dtype=np.int64)
g = gridgen.make_grid('case9241pegase'); c = rh.RedHess(-1); c.load_grid(g); S = c.symbolic()
rp, ci = S['rowptr'], S['colidx']; seg = S['segment']; n = c.n_x
blk = 3
rows = np.flatnonzero(seg == blk)
# bwd local levels (MODE_U): deps = U row (cols > i) in same seg
lv = np.zeros(n, int)
for i in range(n - 1, -1, -1):
    if seg[i] != blk: continue
    row = ci[rp[i]:rp[i+1]]; up = row[row > i]; up = up[seg[up] == blk]
    lv[i] = 1 + lv[up].max() if up.size else 0
nl = lv[rows].max() + 1
dt = np.diff(d[:nl + 1])
for l in range(nl):
    r = rows[lv[rows] == l]
    lens = [(ci[rp[i]:rp[i+1]] > i).sum() for i in r]
    print(l, 'rows', len(r), 'maxlen', max(lens), 'cycles', dt[l] if l < len(dt) else -1)
