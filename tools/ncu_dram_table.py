"""Per-launch DRAM bytes and duration from an ncu --csv metrics list
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum):
    python tools/ncu_dram_table.py <ncu.csv> <out.txt> "<header>"
Writes one row per launch (kernel, grid, duration, DRAM read/write, achieved GB/s)."""
import csv
import sys


def main(path, out, header):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = {}
    order = []
    for r in rows[1:]:
        key = r[ix["ID"]]
        if key not in recs:
            recs[key] = {"name": r[ix["Kernel Name"]], "grid": r[ix.get("Grid Size", 0)] if "Grid Size" in ix else ""}
            order.append(key)
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
                 "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}.get(unit, 1.0)
        recs[key][r[ix["Metric Name"]]] = v * scale
    tot_t = tot_b = 0.0
    with open(out, "w") as f:
        f.write(header + "\n")
        f.write("# launch  us     DRAM_read_MB  DRAM_write_MB  GB/s   kernel\n")
        for k in order:
            d = recs[k]
            t = d.get("gpu__time_duration.sum", 0.0)
            b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            tot_t += t
            tot_b += b
            f.write(f"{k:>6} {t * 1e6:8.1f} {d.get('dram__bytes_read.sum', 0) / 1e6:12.1f} "
                    f"{d.get('dram__bytes_write.sum', 0) / 1e6:13.1f} {b / t / 1e9 if t else 0:7.0f}   {d['name'][:90]}\n")
        f.write(f"# total {tot_t * 1e3:.3f} ms, {tot_b / 1e9:.3f} GB DRAM, {tot_b / tot_t / 1e9:.0f} GB/s "
                f"(serialised, cold-cache per launch)\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
