"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) and an
ncu --page raw --csv capture into the text files kept under profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.txt> "<header line>"
    python tools/ncu_summary.py full <raw.csv> <out.txt> "<header line>"
"""
import collections
import csv
import sys


def launches(path, out, header):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1000.0 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000.0
        tot[r[ki]] += us
        cnt[r[ki]] += 1
    allt = sum(tot.values())
    with open(out, "w") as f:
        f.write(header + "\n")
        f.write(f"# {sum(cnt.values())} launches, {allt/1e3:.3f} ms total (cold-cache, serialised)\n")
        f.write("# launches  total_us  share  kernel\n")
        for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{cnt[k]:8d} {t:10.1f} {100*t/allt:5.1f}%  {k}\n")


KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def full(path, out, header):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w") as f:
        f.write(header + "\n")
        for r in rows[2:]:
            f.write("----\n")
            for k in KEYS:
                if k in idx:
                    f.write(f"  {k:75s} {r[idx[k]]} {units[idx[k]]}\n")
            rd = float(r[idx["dram__bytes_read.sum"]]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[
                units[idx["dram__bytes_read.sum"]]]
            wr = float(r[idx["dram__bytes_write.sum"]]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[
                units[idx["dram__bytes_write.sum"]]]
            us = float(r[idx["gpu__time_duration.sum"]]) * {"usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}[
                units[idx["gpu__time_duration.sum"]]]
            f.write(f"  => DRAM traffic {(rd+wr)/1e9:.4f} GB ({int(rd+wr)} B), {(rd+wr)/us/1e3:.0f} GB/s over the "
                    f"(cold, serialised) launch\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3], sys.argv[4])
