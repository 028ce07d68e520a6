"""Summarise an ncu report: key metrics, stall reasons and SASS op mix per kernel."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if kfilter and kfilter not in name:
        continue
    if name in seen:
        continue
    seen.add(name)
    print("==", name[:110])
    for w in want:
        if w in hdr:
            print(f"   {w} = {r[hdr.index(w)]} {units[hdr.index(w)]}")
    vals = []
    for i, h in enumerate(hdr):
        if "smsp__pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
            try:
                vals.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    print("   stalls:", ", ".join(f"{k}={int(v)}" for v, k in sorted(vals, reverse=True)[:7]))
if kfilter:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kfilter}"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h2 = srows[1]
    ia, isrc, ist, iex = (h2.index("Address"), h2.index("Source"),
                          h2.index("Warp Stall Sampling (All Samples)"), h2.index("Instructions Executed"))
    ops = collections.Counter()
    tot = 0
    seen = set()
    hot = []
    for r in srows[2:]:
        if len(r) <= iex or r[ia] in seen:
            continue
        seen.add(r[ia])
        try:
            ex = int(r[iex] or 0)
            st = int(r[ist] or 0)
        except ValueError:
            continue
        t = r[isrc].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += ex
        tot += ex
        hot.append((st, ex, r[isrc].strip()))
    print("   warp-inst executed:", tot)
    print("   op mix:", ", ".join(f"{k}={v}" for k, v in ops.most_common(14)))
    for h in sorted(hot, reverse=True)[:10]:
        print("   hot:", h)
