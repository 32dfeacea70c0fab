"""Aggregate an ncu launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0][:60]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
for k, v in agg.items():
    print(f"{k:62s} {v[0]:5d} {v[1]/1e3:10.1f} us  {v[1]/1e3/v[0]:9.2f} us/launch {100*v[1]/tot:5.1f}%")
print(len(rows), "launches", round(tot / 1e3, 1), "us")
