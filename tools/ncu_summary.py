"""Summarize an .ncu-rep (raw page) into one line per kernel launch."""
import csv, io, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB", 1e-6),
    ("dram__bytes_write.sum", "MB", 1e-6),
    ("lts__t_bytes.sum", "MB", 1e-6),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%occ", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%sm", 1),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "%mem", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__shared_mem_per_block_dynamic", "smemB", 1),
    ("l1tex__t_sector_hit_rate.pct", "%L1hit", 1),
    ("lts__t_sector_hit_rate.pct", "%L2hit", 1),
]


def unit_scale(unit, want):
    u = unit.strip()
    table = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return table.get(u)


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")[:40]
        parts = [name]
        for m, lab, _ in METRICS:
            if m not in d:
                continue
            v = d[m].replace(",", "")
            u = units[hdr.index(m)]
            try:
                x = float(v)
            except ValueError:
                parts.append(f"{lab}=?")
                continue
            if lab == "us":
                x = x * (unit_scale(u, "s") or 1e-9) * 1e6
            elif lab == "MB":
                x = x * (unit_scale(u, "B") or 1) / 1e6
            parts.append(f"{lab}={x:.1f}")
        print("  ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
