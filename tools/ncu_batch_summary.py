"""Summarize an ncu --set full capture of ONE complete Alg. 2 batch
(tools/prof_hvp.py under --profile-from-start off) into profiles/ncu_summary.json.

    python tools/ncu_batch_summary.py REP.ncu-rep CASE N KIND ROUND [n_x n_p]

Per kernel: duration, DRAM read / write bytes; per stage, its SURVEY.md 8(d)
M2 share (bytes per HVP x N):
  [SpMul + L + U]   (A_L, B_LU, A_U)     reads w, writes z           (n_p + n_x)
  [FoR]             (k_for)              reads z, w; writes y_x, y_p  2 (n_x + n_p)
  [U^T + L^T]       (A_Ut, B_UtLt, A_Lt) reads y_x, writes psi        2 n_x
  [SpMulAdd]        (k_muladd)           reads psi, y_p; writes Hw    n_x + 2 n_p
The k_blk record (mean DRAM bytes per launch, its share of the batch time) and the
block-solve record (k_blk + k_spike DRAM bytes per solve stage, 4 per batch) are
what bench.py reports as roofline.traffic."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for x in r[2:]:
        d = dict(zip(hdr, x))

        def num(m, scale_time=False):
            v = d.get(m, "").replace(",", "")
            u = units[hdr.index(m)] if m in hdr else ""
            try:
                f = float(v)
            except ValueError:
                return None
            if scale_time:
                return f * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}.get(u, 1e-3)
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        res.append({"kernel": d.get("Kernel Name", "?").split("(")[0],
                    "us": num("gpu__time_duration.sum", True),
                    "read": num("dram__bytes_read.sum"), "write": num("dram__bytes_write.sum")})
    return res


def main():
    rep, case, N, kind, rnd = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5]
    nx, npp = (int(sys.argv[6]), int(sys.argv[7])) if len(sys.argv) > 7 else (17036, 2889)
    ks = rows(rep)
    blk = [k for k in ks if k["kernel"] == "k_blk"]
    tot_us = sum(k["us"] for k in ks)
    w = 8.0 * N
    m2 = {"SpMul+L+U": (npp + nx) * w, "FoR": 2 * (nx + npp) * w, "UT+LT": 2 * nx * w, "SpMulAdd": (nx + 2 * npp) * w}
    # stage grouping by launch order: everything before k_for is SpMul + L + U (on a
    # Cartesian batch: plan, L, U0, separator gather + product, k_spike), k_for is
    # FoR, then U^T + L^T until k_muladd
    stages = {"SpMul+L+U": [], "FoR": [], "UT+LT": [], "SpMulAdd": []}
    seen_for = False
    for k in ks:
        n = k["kernel"]
        if n == "k_for":
            seen_for = True
            stages["FoR"].append(k)
        elif n == "k_muladd":
            stages["SpMulAdd"].append(k)
        else:
            stages["UT+LT" if seen_for else "SpMul+L+U"].append(k)
    # the block-solve kernels (k_blk launches and k_spike): 4 solve stages per batch
    solve = [k for k in ks if k["kernel"] in ("k_blk", "k_spike")]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    st = {}
    for s, lst in stages.items():
        us = sum(k["us"] for k in lst)
        dram = sum(k["read"] + k["write"] for k in lst)
        st[s] = {"us": us, "dram_bytes": dram, "m2_bytes": m2[s], "dram_over_m2": dram / m2[s] if m2[s] else None,
                 "m2_frac_of_peak": (m2[s] / (us * 1e-6) / 1e9 / peak) if us else None}
    rec = {
        "round": rnd, "kind": kind, "n_x": nx, "n_p": npp, "N": N, "peak_gbs": peak,
        "kernels": [{k2: (round(v, 3) if isinstance(v, float) else v) for k2, v in k.items()} for k in ks],
        "batch_us_serialized": tot_us,
        "k_blk_dram_bytes_per_launch": sum(k["read"] + k["write"] for k in blk) / max(1, len(blk)),
        "k_blk_time_share": sum(k["us"] for k in blk) / tot_us if tot_us else None,
        "k_blk_m2_bytes_per_launch": (3 * nx + npp) * w / 4.0,
        "solve_kernels": [k["kernel"] for k in solve],
        "solve_dram_bytes_per_stage": sum(k["read"] + k["write"] for k in solve) / 4.0,
        "solve_time_share": sum(k["us"] for k in solve) / tot_us if tot_us else None,
        "stages": st,
        "source": f"ncu --set full --clock-control none --profile-from-start off, tools/prof_hvp.py {case} {N} 3 {kind}",
    }
    rec["k_blk_dram_over_m2"] = rec["k_blk_dram_bytes_per_launch"] / rec["k_blk_m2_bytes_per_launch"]
    rec["solve_dram_over_m2"] = rec["solve_dram_bytes_per_stage"] / rec["k_blk_m2_bytes_per_launch"]
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db = {k: v for k, v in db.items() if isinstance(v, dict) and "kind" in v}   # drop the r01 format
    db[f"{case}:N={N}:{kind}"] = rec
    json.dump(db, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main()
