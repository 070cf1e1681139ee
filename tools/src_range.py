"""Print SASS lines [a, b) (row index) with samples / executions from an ncu source CSV."""
import csv
import gzip
import io
import sys

path, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    lines = f.read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
for idx in range(a, b):
    r = rows[1 + idx]
    print(f"#{idx:5d} {r[si]:>6} {r[ei]:>9} {r[1].strip()[:100]}")
