"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per kernel)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    K = OrderedDict()
    for r in rows[hi + 1:]:
        d = K.setdefault(r[idi], {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[mi]] = v * scale
    return K


if __name__ == "__main__":
    K = load(sys.argv[1])
    tot = sum(v["gpu__time_duration.sum"] for v in K.values())
    by = OrderedDict()
    for k, v in K.items():
        t = v["gpu__time_duration.sum"]
        rd = v.get("dram__bytes_read.sum", 0)
        wr = v.get("dram__bytes_write.sum", 0)
        name = v["name"].split("(")[0][:48]
        by.setdefault(name, [0, 0, 0, 0])
        b = by[name]
        b[0] += t; b[1] += rd; b[2] += wr; b[3] += 1
        print(f"{k:>3} {name:48s} {t:9.3f} ms  rd {rd/1e9:7.3f} GB  wr {wr/1e9:7.3f} GB  {((rd+wr)/1e6/t) if t else 0:8.1f} GB/s")
    print(f"total {tot:.3f} ms")
    for name, b in by.items():
        print(f"{name:48s} x{b[3]:<3} {b[0]:9.3f} ms ({100*b[0]/tot:5.1f}%)  {(b[1]+b[2])/1e9:7.2f} GB")
