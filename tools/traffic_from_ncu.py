"""Per-program DRAM traffic from an ncu launch list of tools/prof_run.py:
sum dram__bytes_read.sum + dram__bytes_write.sum over the captured propagation
kernels and divide by the number of programs run.  Writes the JSON that
bench.py reports as roofline.traffic.
usage: python tools/traffic_from_ncu.py launches.csv n_programs config dtype batch [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as n  # noqa: E402

path, runs, config, dtype, batch = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
d = n.load(path)
rd = sum(n.val(m, "dram__bytes_read.sum") for m in d.values())
wr = sum(n.val(m, "dram__bytes_write.sum") for m in d.values())
t = sum(n.val(m, "gpu__time_duration.sum") for m in d.values())
doc = {"bytes_per_launch": int((rd + wr) / runs), "read_bytes": int(rd / runs), "write_bytes": int(wr / runs),
       "ncu_us_per_program": round(t / runs, 1), "kernels_per_program": len(d) // runs,
       "source": f"ncu launch list {os.path.basename(path)} ({runs} programs, cold-cache serialised replay)"}
out = sys.argv[6] if len(sys.argv) > 6 else os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                                          f"traffic_{config}_{dtype}_b{batch}.json")
with open(out, "w") as f:
    json.dump(doc, f, indent=1)
print(json.dumps(doc))
