"""Summarise an ncu launch list (--metrics gpu__time_duration.sum CSV) and an ncu --set full
report into a small markdown file for profiles/.

usage: python tools/ncu_summary.py LAUNCHES.csv REPORT.ncu-rep OUT.md [title]
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "pcie__read_bytes.sum.per_second",
        "pcie__write_bytes.sum.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / tot:.3f} | {sum(v) / len(v) / 1e3:.1f} |")
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    ix = [(k, h.index(k)) for k in KEYS if k in h]
    out = ["| kernel | " + " | ".join(f"{k} ({units[i]})" for k, i in ix) + " |",
           "|---" * (len(ix) + 1) + "|"]
    for row in r[2:]:
        out.append(f"| {row[h.index('Kernel Name')].split('(')[0]} | " + " | ".join(row[i] for _, i in ix) + " |")
    return out


if __name__ == "__main__":
    lc, rep, outp = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else "ncu summary"
    lines = [f"# {title}", "", "## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; "
             "cold-cache, serialised: compare shares)", ""] + launches(lc) + \
            ["", "## ncu --set full (one launch each)", ""] + full(rep) + [""]
    open(outp, "w").write("\n".join(lines))
    print("\n".join(lines))
