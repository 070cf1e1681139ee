"""profiles/traffic.json: dram read + write bytes per launch for every kernel in
the given ncu raw-page CSVs (first capture of each kernel name wins)."""
import csv
import io
import json
import sys


def main(out, paths):
    res = {}
    for p in paths:
        rows = list(csv.reader(io.StringIO(open(p).read())))
        hdr = rows[0]
        ki = hdr.index("Kernel Name")
        ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        units = rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[2:]:
            name = r[ki].split("(")[0].split("::")[-1]
            if name in res:
                continue
            rd = float(r[ri].replace(",", "")) * scale.get(units[ri], 1)
            wr = float(r[wi].replace(",", "")) * scale.get(units[wi], 1)
            res[name] = int(rd + wr)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
