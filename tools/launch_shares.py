"""Per-kernel share of the last timed step in an ncu launch list
(gpu__time_duration.sum CSV): the launches after the previous step's last
stress_kernel up to and including the last stress_kernel."""
import collections
import csv
import re
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))
        if r["Metric Name"] == "gpu__time_duration.sum"]
stress = [i for i, r in enumerate(rows) if "stress_kernel" in r["Kernel Name"]]
end = stress[-1]
prev = [i for i in stress if i < end]
# step boundary: the previous step's last stress launch (followed by a solver kernel)
start = 0
for i in reversed(prev):
    nxt = rows[i + 1]["Kernel Name"]
    if not any(k in nxt for k in ("stress_kernel", "gemm_nt_f64", "gemm_seg_f64", "scatter_vec", "sym_fine", "sym_panel", "k6_face")):
        start = i + 1
        break
acc = collections.OrderedDict()
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows[start:end + 1]:
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("tsvb200::", "").replace("void ", "")
    us = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    a = acc.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in acc.values())
print("kernel,launches,total_us,mean_us,share")
for k, (n, us) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k},{n},{us:.1f},{us / n:.2f},{us / tot:.3f}")
print(f"TOTAL,{sum(v[0] for v in acc.values())},{tot:.1f},,1.000")
