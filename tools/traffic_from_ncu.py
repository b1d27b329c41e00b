"""Per-program DRAM traffic from an ncu launch list of tools/prof_run.py:
sum dram__bytes_read.sum + dram__bytes_write.sum over the captured propagation
kernels and divide by the number of programs run.  Writes the JSON that
bench.py reports as roofline.traffic.
usage: python tools/traffic_from_ncu.py launches.csv n_programs config dtype batch [out.json]
(n_programs is recomputed from the ev_fill launches; the argument is kept for old callers)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as n  # noqa: E402

path, runs, config, dtype, batch = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
d = n.load(path)
# one step = evidence masks (ev_fill, ev_zero) + the propagation program + the
# normalize kernel: count from the first ev_fill on (state creation fills the
# arenas once, before any step) and divide by the number of steps seen
items = list(d.items())
first = next(i for i, ((k, name), m) in enumerate(items) if name.startswith("ev_fill"))
steps = [(k, m) for (k, name), m in items[first:]]
runs = sum(1 for (k, name), m in items[first:] if name.startswith("ev_fill"))
rd = sum(n.val(m, "dram__bytes_read.sum") for _, m in steps)
wr = sum(n.val(m, "dram__bytes_write.sum") for _, m in steps)
t = sum(n.val(m, "gpu__time_duration.sum") for _, m in steps)
d = dict(steps)
doc = {"bytes_per_launch": int((rd + wr) / runs), "read_bytes": int(rd / runs), "write_bytes": int(wr / runs),
       "ncu_us_per_program": round(t / runs, 1), "kernels_per_program": len(d) // runs,
       "source": f"ncu launch list {os.path.basename(path)} ({runs} programs, cold-cache serialised replay)"}
out = sys.argv[6] if len(sys.argv) > 6 else os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                                          f"traffic_{config}_{dtype}_b{batch}.json")
with open(out, "w") as f:
    json.dump(doc, f, indent=1)
print(json.dumps(doc))
