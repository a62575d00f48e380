import numpy as np
d = np.fromfile("gpurun_out/kseg_rows.bin", dtype=np.int64).reshape(-1, 2)
# rows of warp 0 (code < 100000)
for q in range(len(d) - 1):
    if d[q, 0] == 0 or d[q + 1, 0] == 0: continue
    code = d[q, 1]; w = code // 100000; sl = (code % 100000) // 1000; ne = code % 1000
    code2 = d[q + 1, 1]; w2 = code2 // 100000
    if w == 0 and w2 == 0:
        print(q, "sl", sl, "entries", ne, "cycles", d[q + 1, 0] - d[q, 0])
