"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes] per launch):
per-kernel totals and shares, and every launch of a kernel matching --kernel."""
import argparse
import csv
import json
from collections import defaultdict


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = {h: i for i, h in enumerate(rows[0])}
    launches = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = int(r[hdr["ID"]])
        names[lid] = r[hdr["Kernel Name"]]
        launches[lid][r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
    return names, launches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--kernel", default="box_copy")
    args = ap.parse_args()
    names, launches = load(args.csv)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for lid, m in launches.items():
        short = names[lid].split("(")[0][-60:]
        tot[short] += m.get("gpu__time_duration.sum", 0.0)
        cnt[short] += 1
    all_ns = sum(tot.values())
    summary = [{"kernel": k, "launches": cnt[k], "ms": round(v / 1e6, 3), "share": round(v / all_ns, 4)}
               for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    sel = [{"id": lid, **{k: int(v) for k, v in m.items()}} for lid, m in sorted(launches.items())
           if args.kernel in names[lid]]
    print(json.dumps({"kernels": summary, "selected": sel}, indent=1))


if __name__ == "__main__":
    main()
