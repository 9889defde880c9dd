# lone-frame kernel durations (cfg2 S=1) and the 64-frame chain merge, ncu launch lists
for w in cfg2 seq64; do
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/r02bq_${w}.csv python tools/prof_frames.py $w > /dev/null 2>&1
done
python - <<'PY'
import csv, collections
for w in ("cfg2", "seq64"):
    rows = list(csv.DictReader(l for l in open(f"gpurun_out/r02bq_{w}.csv") if l.startswith('"')))
    d = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            d[r["Kernel Name"][:60]].append(float(r["Metric Value"].replace(",", "")))
    print("==", w)
    for k, v in d.items():
        v = v[-3:]
        print(f"  {k:60s} n={len(v)} last3 mean {sum(v)/len(v):9.1f} ns")
PY
