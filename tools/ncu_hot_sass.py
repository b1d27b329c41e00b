"""Top SASS lines by warp-stall samples for one launch of an ncu report.
usage: python tools/ncu_hot_sass.py report.ncu-rep launch_index [top]"""
import csv
import io
import subprocess
import sys


def main(path, idx, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--launch-skip", str(idx),
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    print(rows[0][1])
    hdr = rows[1]
    ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[ia].startswith("0x")]
    tot = sum(int(r[ist] or 0) for r in body)
    print("total samples", tot)
    for n, r in enumerate(body):
        r.append(n)
    for r in sorted(body, key=lambda r: -int(r[ist] or 0))[:top]:
        print(f"{r[-1]:5d} {int(r[ist]):7d} {100*int(r[ist])/tot:5.1f}%  {r[isrc].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
