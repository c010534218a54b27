"""Write profiles/attn_traffic.json from ncu launch lists (dram__bytes_read.sum +
dram__bytes_write.sum per launch of the attention kernel), one entry per config.

    python tools/attn_traffic.py CONFIG KERNEL_NAME launches.csv [CONFIG KERNEL_NAME launches.csv ...]

KERNEL_NAME is the library's ba_attention_kernel_name (what bench.py reports); the
SASS kernel is matched by its template name (attn_pp_kernel / attn_sm100_kernel)."""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
SASS = {"attn_sm100_tcgen05_pp": "attn_pp_kernel", "attn_sm100_tcgen05_pp64": "attn_pp_kernel",
        "attn_sm100_tcgen05_dual64": "attn_sm100_kernel", "attn_sm100_tcgen05": "attn_sm100_kernel"}


def per_launch(path, sass):
    per = {}
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if sass not in d["Kernel Name"]:
                continue
            m = per.setdefault(int(d["ID"]), {"name": d["Kernel Name"].split("(")[0]})
            m[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
    return list(per.values())


def main(argv):
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "attn_traffic.json")
    entries = []
    for i in range(0, len(argv), 3):
        cfg, kname, path = argv[i:i + 3]
        launches = [m for m in per_launch(path, SASS[kname]) if "dram__bytes_read.sum" in m]
        if not launches:
            raise SystemExit(f"no {SASS[kname]} launches with DRAM metrics in {path}")
        rd = sum(m["dram__bytes_read.sum"] for m in launches) / len(launches)
        wr = sum(m["dram__bytes_write.sum"] for m in launches) / len(launches)
        entries.append({"config": cfg, "kernel": kname, "sass_kernel": launches[0]["name"],
                        "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                        "launches": len(launches), "source": f"{os.path.basename(path)} (ncu dram__bytes_read.sum + "
                                                             "dram__bytes_write.sum, mean over launches)"})
    json.dump({"entries": entries}, open(out, "w"), indent=1)
    print(json.dumps(entries, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
