"""Summarise `ncu --page raw --csv` exports: one row per profiled launch with the metrics
the roofline discussion uses.  usage: python tools/ncu_summary.py raw.csv [...]"""
import csv, sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps act %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    kn = ix.get("Kernel Name")
    print("| kernel | " + " | ".join(f"{c[1]} ({units[ix[c[0]]]})" if c[0] in ix else c[1] for c in COLS) + " |")
    print("|---" * (len(COLS) + 1) + "|")
    for r in rows[2:]:
        name = r[kn][:34] if kn is not None else "?"
        vals = []
        for c, _ in COLS:
            v = r[ix[c]] if c in ix else ""
            try:
                f = float(v.replace(",", ""))
                v = f"{f:.4g}"
            except ValueError:
                pass
            vals.append(v)
        print(f"| {name} | " + " | ".join(vals) + " |")
