"""Per-source-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr = None, None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 6:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:70])
    if cur is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    a = agg[cur[:2]]
    a[0] += s
    a[3] = cur[2]
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
            try: a[2][k[6:]] += int(v)
            except ValueError: pass
tot = sum(v[0] for v in agg.values())
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = ", ".join(f"{k} {c}" for k, c in v[2].most_common(3))
    print(f"{100*v[0]/tot:5.1f}% {key[0]}:{key[1]:<4d} {v[3]:70s} | {st}")
