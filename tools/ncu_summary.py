"""Summarise ncu output for profiles/: launch lists (per-kernel device time)
and --set full captures (SOL, occupancy, stalls, tensor / DRAM counters).

    python tools/ncu_summary.py launches <launches.csv>
    python tools/ncu_summary.py full <report.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[mi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total ms':>10} {'ms/launch':>10} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:8d} {t:10.3f} {t / c:10.3f} {100 * t / tot:5.1f}%  {k}")


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def full(path, kid=None):
    """Summary of one kernel of a --set full report (kid: its ID, default the first)."""
    det = list(csv.reader(io.StringIO(ncu([path, "--page", "details", "--csv"]))))
    h = det[0]
    if kid is not None:
        ii = h.index("ID")
        det = [h] + [r for r in det[1:] if len(r) > ii and r[ii] == str(kid)]
    print("kernel:", dict(zip(h, det[1])).get("Kernel Name", "")[:120])
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Compute (SM) Throughput",
            "Issue Slots Busy", "Executed Ipc Active", "Achieved Active Warps Per SM",
            "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
            "Avg. Active Threads Per Warp", "Registers Per Thread", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block"}
    for row in det[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in keep:
            print(f"  {d['Metric Name']:<40} {d['Metric Value']:>14} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(ncu([path, "--page", "raw", "--csv"]))))
    rh = raw[0]
    rows = raw[2:] if len(raw) > 2 else raw[1:]
    if kid is not None and "ID" in rh:
        rows = [r for r in rows if r[rh.index("ID")] == str(kid)] or rows
    rv = rows[0]
    for a, b in zip(rh, rv):
        if a in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                 "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                 "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
                 "gpu__time_duration.sum", "launch__registers_per_thread",
                 "sm__warps_active.avg.pct_of_peak_sustained_active"):
            print(f"  {a:<60} {b}")
    src = list(csv.reader(io.StringIO(ncu([path, "--page", "source", "--csv",
                                           "--print-source", "sass"]))))
    sh = src[1]
    cols = [(i, c) for i, c in enumerate(sh) if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    top = []
    ie, isrc, iall = sh.index("Instructions Executed"), sh.index("Source"), \
        sh.index("Warp Stall Sampling (All Samples)")
    for r in src[2:]:
        if len(r) <= ie:
            continue
        for i, c in cols:
            try:
                agg[c] += float(r[i] or 0)
            except ValueError:
                pass
        try:
            top.append((float(r[iall] or 0), r[isrc].strip()))
        except ValueError:
            pass
    t = sum(agg.values()) or 1
    print("  stall reasons (share of samples):")
    for k, v in agg.most_common(8):
        print(f"    {k:<28} {100 * v / t:5.1f}%")
    ts = sum(x[0] for x in top) or 1
    print("  top SASS by stall samples:")
    for s, line in sorted(top, reverse=True)[:12]:
        print(f"    {100 * s / ts:5.1f}%  {line[:100]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
