"""Print ms/iter and work counters of trace_run.py outputs: python tools/cmp_traces.py FILE..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable:", str(e)[:80]); continue
    st = d.get("stats", {})
    tv = max(1, st.get("tile_visits", 0))
    print(f"{f:55s} {d['ms_per_iter']:.4f} ms/iter  visits {st.get('tile_visits', 0)}  batch {st.get('batch_tiles', 0)}"
          f"  pairs {st.get('pairs', 0)}")
