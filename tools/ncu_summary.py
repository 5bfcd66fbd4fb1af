#!/usr/bin/env python
"""Summarise ncu outputs for profiles/.

  tools/ncu_summary.py launches <launches.csv>      per-kernel share of device time
  tools/ncu_summary.py report <file.ncu-rep>...     key metrics of a --set full capture
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("wrmg::<unnamed>::", "")


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"]) + " grid" + r["Grid Size"]
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            v *= 1e3
        elif r["Metric Unit"] == "ms":
            v *= 1e6
        tot[k] += v
        cnt[k] += 1
    all_ns = sum(tot.values())
    print(f"# {len(rows)} launches, {all_ns / 1e6:.3f} ms total device time (cold-cache, serialised)")
    print(f"{'share':>7} {'ms':>10} {'launches':>8} {'us/launch':>10}  kernel")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / all_ns:6.2f}% {v / 1e6:10.3f} {cnt[k]:8d} {v / cnt[k] / 1e3:10.2f}  {k}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for val in rows[2:]:
        d = dict(zip(hdr, val))
        print(f"## {short(d.get('Kernel Name', '?'))} grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {units[hdr.index(k)]}")
        st = sorted(((k, float(d[k] or 0)) for k in hdr
                     if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")),
                    key=lambda kv: -kv[1])[:6]
        print("  top stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}"
                                                          for k, v in st))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
