"""Summarise ncu captures into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py <report.ncu-rep> [...]      -> markdown table on stdout
  python tools/ncu_summary.py --launches <launches.csv>   -> per-kernel share table
  python tools/ncu_summary.py --raw <raw.csv> [...]        -> the same table from `ncu -i X --page raw --csv`
                                                              exported on the GPU box
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__cluster_dim_x",
    "launch__registers_per_thread",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "lts__t_sectors_srcunit_tex_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_lookup_miss.sum",
    "lts__t_sectors_srcunit_tex_evict_last_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_evict_last_lookup_miss.sum",
    "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second",
]


def report(path, raw_text=None):
    out = raw_text if raw_text is not None else subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                                                               capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    rows = rows[start:]
    hdr, units = rows[0], rows[1]
    print(f"### {path}\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"kernel `{name[:90]}`\n\n| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
                agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {sum(v)/tot:.1%} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--raw":
        for p in sys.argv[2:]:
            report(p, open(p).read())
    else:
        for p in sys.argv[1:]:
            report(p)
