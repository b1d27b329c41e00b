"""Top launches and per-kernel totals of the last program in an ncu launch list (tools/gpu_list_one.sh)."""
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_summary as n  # noqa: E402

d = n.load(sys.argv[1])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
items = list(d.items())
idx = [i for i, ((k, name), m) in enumerate(items) if name.startswith("ev_fill")]
last = items[idx[-1]:]
rows, agg = [], {}
for (k, name), m in last:
    t = n.val(m, "gpu__time_duration.sum")
    rd = n.val(m, "dram__bytes_read.sum") / 1e9
    wr = n.val(m, "dram__bytes_write.sum") / 1e9
    g = m.get("launch__grid_size", ("", ""))[1]
    rows.append((t, k, name.split("(")[0].replace("void ", ""), rd, wr, g))
    a = agg.setdefault(name.split("(")[0].replace("void ", ""), [0, 0, 0])
    a[0] += t
    a[1] += rd + wr
    a[2] += 1
print("program sum %.0f us, %d launches, DRAM %.1f GB" % (sum(r[0] for r in rows), len(rows), sum(r[3] + r[4] for r in rows)))
for r in sorted(rows, reverse=True)[:top]:
    print("  %8.1f us %4d %-50s rd %6.2f wr %6.2f GB %5.2f TB/s grid %s" % (r[0], r[1], r[2][:50], r[3], r[4], (r[3] + r[4]) / r[0] * 1e3, r[5]))
for k, (t, b, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print("  %-50s %3d %8.0f us %6.1f GB %5.2f TB/s" % (k[:50], c, t, b, b / t * 1e3))
