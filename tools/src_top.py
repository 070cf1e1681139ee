"""Top SASS lines by warp-stall samples from an ncu source-page CSV (gz ok)."""
import csv
import gzip
import io
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    lines = f.read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
si, ni, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)"), hdr.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[1:]):
    try:
        data.append((int(r[si]), int(r[ni]), int(r[ei]), idx, r[0][-5:], r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", sum(d[2] for d in data))
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:7d} {100*d[0]/tot:5.1f}% ni={d[1]:6d} ex={d[2]:9d} #{d[3]:5d} {d[5][:90]}")
