"""Summary of one ncu --set full capture of a sweep kernel (profiles/*_ncu_full.txt):
time, DRAM bytes, issue activity, shared-memory wavefronts/conflicts, stall
reasons, op mix and the hottest SASS lines. With --traffic also rewrites
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).
Usage: ncu_diag_summary.py report.ncu-rep [--traffic] [--kernel REGEX]"""
import csv, io, json, os, subprocess, sys
from collections import Counter

rep = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import re
kre = re.compile(sys.argv[sys.argv.index("--kernel") + 1]) if "--kernel" in sys.argv else None
run = lambda *a: subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, units = rows[0], rows[1]
r = next(x for x in rows[2:] if kre is None or kre.search(x[h.index("Kernel Name")]))
d = dict(zip(h, r))
u = dict(zip(h, units))
num = lambda k: float(d[k].replace(",", ""))
mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
name = d["Kernel Name"]
out = [f"== {name}"]
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
          "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in d:
        out.append(f"   {k} = {d[k]} {u[k]}")
st = sorted(((num(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in h
             if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
             and d[k].replace(",", "").replace(".", "").isdigit()), reverse=True)
out.append("   stalls (pc samples): " + ", ".join(f"{k}={int(v)}" for v, k in st[:8] if v > 0))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
sections, cur = [], None
for row in src:  # one section per kernel: ["Kernel Name", name], header, rows
    if row and row[0] == "Kernel Name":
        cur = [row[1] if len(row) > 1 else "", None, []]
        sections.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
sec = next(x for x in sections if kre is None or kre.search(x[0]))
sh = sec[1]
sd = [row for row in sec[2] if len(row) == len(sh)]
ix = {k: i for i, k in enumerate(sh)}
f = lambda row, k: float(row[ix[k]].replace(",", "") or 0) if k in ix and row[ix[k]] else 0.0
ops, wf, ex = Counter(), Counter(), Counter()
for row in sd:
    toks = row[ix["Source"]].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    ops[op] += f(row, "Instructions Executed")
    wf[op] += f(row, "L1 Wavefronts Shared")
    ex[op] += f(row, "L1 Wavefronts Shared Excessive")
out.append("   op mix: " + ", ".join(f"{k}={int(v)}" for k, v in ops.most_common(14)))
out.append("   shared wavefronts by op: " + ", ".join(f"{k}={int(v)} (excess {int(ex[k])})"
                                                     for k, v in wf.most_common(5) if v))
hot = sorted(sd, key=lambda row: -f(row, "Warp Stall Sampling (All Samples)"))[:10]
for row in hot:
    out.append(f"   hot: {int(f(row, 'Warp Stall Sampling (All Samples)'))} samples, "
               f"{int(f(row, 'Instructions Executed'))} exec  {row[ix['Source']].strip()[:70]}")
print("\n".join(out))
if "--traffic" in sys.argv:
    # --windows K: the capture is one persistent launch over K windows (per step = / K)
    kw = int(sys.argv[sys.argv.index("--windows") + 1]) if "--windows" in sys.argv else 1
    rd = num("dram__bytes_read.sum") * mb[u["dram__bytes_read.sum"]] * 1e6 / kw
    wr = num("dram__bytes_write.sum") * mb[u["dram__bytes_write.sum"]] * 1e6 / kw
    alg = 8 * 1_000_000 * 12 + 1_000_000 * 12 // 8 + 8 * 64 * 12 + 16 * 64
    json.dump({"source": f"{os.path.basename(rep)} (ncu --set full --clock-control none, "
                         + ("tools/profile_windows.py" if kw > 1 else "tools/profile_sweep.py diagonal") + ")",
               "kernel": name + (f" (one launch over {kw} config-4 windows; bytes per window)" if kw > 1
                                 else " (the whole config-4 sweep is this one launch)"),
               "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
               "sweep_dram_bytes_per_step": int(rd + wr), "algorithmic_bytes_per_step": alg,
               "note": "read = 96 MB f64 scores + 4 MB u32 correctness rows (4 B/sample vs the "
                       "bit-packed 1.5 B/sample algorithmic figure); write = per-CTA count "
                       f"merges + results. traffic/algorithmic = {(rd + wr) / alg:.3f}"},
              open(os.path.join(root, "profiles", "ncu_traffic.json"), "w"), indent=1)
