"""One line per captured kernel: time, DRAM GB/s (and % of the measured peak),
tensor-pipe utilisation, issue activity. Usage: ncu_kernels_summary.py report.ncu-rep"""
import csv, io, json, os, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6450.0
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
bscale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def val(r, k):
    i = h.index(k)
    return float(r[i].replace(",", "")), units[i]


for r in rows[2:]:
    name = r[h.index("Kernel Name")][:70]
    t, tu = val(r, "gpu__time_duration.sum")
    t *= scale.get(tu, 1.0)
    rd, ru = val(r, "dram__bytes_read.sum")
    wr, wu = val(r, "dram__bytes_write.sum")
    mb = rd * bscale.get(ru, 1.0) + wr * bscale.get(wu, 1.0)
    gbs = mb * 1e-3 / (t * 1e-6) if t else 0.0
    tens = r[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")] \
        if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in h else "n/a"
    iss = r[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]
    grid = r[h.index("launch__grid_size")]
    print(f"{name:70s} {t:9.2f} us  grid {grid:>6}  DRAM {mb:8.2f} MB {gbs:7.0f} GB/s "
          f"({100 * gbs / peak:5.1f}% of {peak:.0f})  tensor-pipe {tens:>6}%  issue {iss}%")
