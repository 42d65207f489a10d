"""Collect per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and, when captured,
warp-instructions (smsp__inst_executed.sum) from single-pass ncu metric CSVs into
profiles/ncu_traffic_r02.json, which bench.py reads for the roofline `traffic` field.

usage: python tools/ncu_traffic.py out.json key=capture.csv [key=capture.csv ...]
Each value is the mean over the launches in that capture."""
import csv
import json
import os
import sys
from collections import defaultdict


# ncu auto-scales units in CSV output; bring bytes to bytes and durations to ns
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "s": 1e9, "second": 1e9}


def parse(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iid, im, iu, iv = h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    per = defaultdict(dict)
    for r in rows[1:]:
        per[r[iid]][r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    return list(per.values())


def main():
    out = sys.argv[1]
    res = {}
    if os.path.exists(out):
        with open(out) as f:
            res = json.load(f)
    for kv in sys.argv[2:]:
        key, path = kv.split("=", 1)
        if not os.path.exists(path):
            print("missing", path)
            continue
        launches = parse(path)
        if not launches:
            print("no launches in", path)
            continue
        n = len(launches)
        byts = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in launches) / n
        ent = {"bytes": byts, "launches": n, "source": os.path.basename(path)}
        if all("smsp__inst_executed.sum" in l for l in launches):
            ent["inst"] = sum(l["smsp__inst_executed.sum"] for l in launches) / n
        if all("gpu__time_duration.sum" in l for l in launches):
            ent["ncu_ms"] = sum(l["gpu__time_duration.sum"] for l in launches) / n / 1e6
        loc = [l.get("l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", 0)
               + l.get("l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum", 0) for l in launches]
        if any(loc):
            ent["local_bytes"] = sum(loc) / n
        res[key] = ent
        print(key, ent)
    res["_note"] = ("per-launch means from single-pass ncu metric captures (--clock-control none) of the "
                    "same launch configuration bench.py times, at this round's code; see each 'source'")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
