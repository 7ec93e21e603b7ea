"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV).

    python tools/launch_summary.py launches.csv [out.json]
ncu times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in data:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        us = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        tot[name] = tot.get(name, 0.0) + us
        cnt[name] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "total_us": round(v, 1), "mean_us": round(v / cnt[k], 2),
                "share": round(v / s, 4)} for k, v in sorted(tot.items(), key=lambda x: -x[1])}


if __name__ == "__main__":
    out = summarise(sys.argv[1])
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)
