"""Group an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by
kernel name: launches, total us, share. Usage: launch_list_summary.py list.csv [top]"""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ui = h.index("Metric Unit")
idi = h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[idi]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    names[r[idi]] = r[ki]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bsc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Kbyte ": 1e-3}
for i, m in per.items():
    t, u = m["gpu__time_duration.sum"]
    t *= scale.get(u, 1.0)
    mb = sum(v * bsc.get(uu, 1.0) for k, (v, uu) in m.items() if k.startswith("dram__bytes"))
    n = names[i][:90]
    tot[n][0] += 1
    tot[n][1] += t
    tot[n][2] += mb
all_t = sum(v[1] for v in tot.values())
print(f"total {all_t:.1f} us over {sum(v[0] for v in tot.values())} launches")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
has_bytes = any(v[2] > 0 for v in tot.values())  # only when the list carries dram__bytes
for n, (c, t, mb) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
    bw = f"{mb * 1e-3 / max(t * 1e-6, 1e-12):7.0f} GB/s  " if has_bytes else ""
    print(f"{t:9.1f} us {100*t/all_t:5.1f}% x{c:3d}  {bw}{n}")
