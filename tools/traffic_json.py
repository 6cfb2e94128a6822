"""Fold an ncu --csv traffic list (dram__bytes_read/write + duration per
launch, one bbml_pnn_train call and one bbml_lm_train call of
`tools/prof.py --precision 64 --restarts 32 --reps 1`) into
profiles/r02_traffic.json, the per-call DRAM bytes bench.py reports as
roofline.traffic.

usage: python tools/traffic_json.py gpurun_out/final/traffic.csv profiles/r02_traffic.csv
"""
import csv
import io
import json
import shutil
import sys
from collections import OrderedDict


def main(src, dst_csv):
    text = open(src).read()
    body = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(body)))
    per = OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        key = "pnn_fp64" if name.startswith("void pnn_") else "lm"
        k = per.setdefault(key, OrderedDict()).setdefault(name, {})
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1.0, "us": 1e-3,
                 "ns": 1e-6, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(r["Metric Unit"], 1.0)
        k[r["Metric Name"]] = k.get(r["Metric Name"], 0.0) + v * scale
    out = {}
    call = {"pnn_fp64": "bbml_pnn_train", "lm": "bbml_lm_train"}
    for key, ks in per.items():
        tot = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
                  for m in ks.values())
        parts = ", ".join(f"{n[5:]} {m.get('dram__bytes_read.sum', 0) / 1e6:.1f}+"
                          f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} MB" for n, m in ks.items())
        out[key] = {"bytes_per_launch": tot, "workload": "suite16",
                    "report": f"{dst_csv} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                              f"over every launch of one {call[key]} call, suite16 x32 FP64: {parts})",
                    "kernels": ks}
    shutil.copy(src, dst_csv)
    json.dump(out, open(dst_csv[:-4] + ".json", "w"), indent=1)
    print(json.dumps({k: v["bytes_per_launch"] for k, v in out.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
