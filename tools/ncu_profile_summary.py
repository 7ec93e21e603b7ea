"""profiles/ncu_summary.json from the raw ncu exports of tools/refresh_profiles.sh:
per workload and step kernel, the DRAM bytes of one launch (the `traffic` of
bench.py's roofline), its duration (ncu: cold-cache, serialised), warps active,
registers and the top stall reasons.

    python tools/ncu_profile_summary.py gpurun_out/prof > profiles/ncu_summary.json
"""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarise  # noqa: E402

WORKLOADS = {"full_240_raw.csv": "240^3", "full_512_raw.csv": "512^3",
             "full_1000_raw.csv": "1000^3", "full_512_r2_raw.csv": "512^3 r2",
             "full_512_r8_raw.csv": "512^3 r8", "full_cpml_240_raw.csv": "240^3 cpml_fused"}


def kname(k):
    if "k_inner" in k:
        return "inner"
    if "k_zslab" in k:
        return "inner"  # the column kernel serves the inner box at r > 4
    if "k_bnd" in k:
        return "boundary"
    if "k_cpml" in k:
        return "cpml"
    m = re.search(r"k_p1<\s*\d+,\s*\d+,\s*(\w+)\s*>", k)
    if m:
        return "pass1_z" if m.group(1) in ("1", "true") else "pass1_xy"
    return k


def nbytes(v):
    """'1.43 Gbyte' -> bytes (each metric carries its own unit)."""
    t = str(v).split()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(t[-1] if len(t) > 1 else "", 1)
    return float(t[0].replace(",", "")) * scale


def main(d):
    out = {}
    for fn, wl in WORKLOADS.items():
        p = Path(d) / fn
        if not p.exists():
            continue
        rows = summarise(str(p))
        ent = {}
        for r in rows:
            name = kname(r.get("Kernel Name", ""))
            rd = nbytes(r.get("dram__bytes_read.sum", "0"))
            wr = nbytes(r.get("dram__bytes_write.sum", "0"))
            scale = 1.0
            ent[name] = {"kernel": r.get("Kernel Name"),
                         "dram_bytes_per_launch": (rd + wr) * scale,
                         "duration": r.get("gpu__time_duration.sum"),
                         "warps_active": r.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                         "regs": r.get("launch__registers_per_thread"),
                         "grid": r.get("launch__grid_size"), "block": r.get("launch__block_size"),
                         "dram_throughput": r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                         "stalls": r.get("top_stalls_per_issue")}
        out[wl] = ent
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof")
