#!/bin/bash
# Per-launch durations of the Schwarz iteration kernels (ncu), printed per kernel.
cfg=${1:-3}
python tools/prof_as.py $cfg > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/as_list.csv python tools/prof_as.py $cfg > /dev/null 2>&1
python - <<PY
import csv,collections,re
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/as_list.csv") if not l.startswith("==")) if r["Metric Name"]=="gpu__time_duration.sum"]
acc=collections.OrderedDict()
for r in rows:
    n=re.sub(r"\(.*","",r["Kernel Name"]).replace("tsvb200::","").replace("void ","")
    acc.setdefault(n,[]).append(float(r["Metric Value"].replace(",",""))/1000)
tot=0
for n,v in acc.items():
    real=[x for x in v if x>8.0] if len(v)>=8 else []
    if real:
        m=sorted(real)[len(real)//2]; tot+=m
        print(f"{n[:60]:60s} median {m:8.1f} us  n={len(real)}")
print("sum of medians", round(tot,1))
PY
