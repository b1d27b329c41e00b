"""Summarise an ncu --csv launch list: per kernel launch id, name, metrics."""
import csv
import sys
from collections import OrderedDict

def load(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    out = OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        out.setdefault(key, {})[d["Metric Name"]] = (d["Metric Unit"], d["Metric Value"])
    return out

def val(m, name):
    u, v = m.get(name, ("", "0"))
    v = float(v.replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "Kbyte": 1e3, "KB": 1e3, "MB": 1e6, "GB": 1e9, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return v * scale.get(u, 1.0)

if __name__ == "__main__":
    data = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    tot = 0
    print(f"{'id':>4} {'kernel':40} {'us':>10} {'dramRd MB':>10} {'dramWr MB':>10} {'L2 MB':>10} {'GB/s':>8}")
    for (i, name), m in data.items():
        if i < skip:
            continue
        t = val(m, "gpu__time_duration.sum")
        rd = val(m, "dram__bytes_read.sum") / 1e6
        wr = val(m, "dram__bytes_write.sum") / 1e6
        l2 = val(m, "lts__t_bytes.sum") / 1e6
        tot += t
        print(f"{i:4d} {name[:40]:40} {t:10.1f} {rd:10.2f} {wr:10.2f} {l2:10.1f} {(rd+wr)*1e6/max(t,1e-9)/1e3:8.0f}")
    print("total us", tot)
