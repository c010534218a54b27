"""Summarise an ncu --csv launch list: per-kernel average time and DRAM traffic."""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "nsecond": 1e-3}


def summarise(path, skip_first=0):
    rows = [r for r in csv.reader(open(path))]
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"].split("(")[0][:60])
            per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
    agg = collections.OrderedDict()
    for (i, n), m in per.items():
        if i < skip_first:
            continue
        a = agg.setdefault(n, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    out = []
    tot = sum(a[1] for a in agg.values())
    for n, (c, t, rd, wr) in agg.items():
        out.append(f"{c:3d} x {t / c:9.1f} us  share {100 * t / tot:5.1f}%  dram rd {rd / c / 1e6:9.1f} MB wr {wr / c / 1e6:8.1f} MB "
                   f"= {(rd + wr) / c / (t / c * 1e-6) / 1e9:6.0f} GB/s  {n}")
    out.append(f"total {tot:.1f} us")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0))
