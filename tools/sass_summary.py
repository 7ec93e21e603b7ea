"""SASS evidence for the built library: per kernel (mangled name) the static
counts of TMA loads (UTMALDG), 128-bit shared loads (LDS.128), 128-bit global
stores (STG.E.128), packed FP32 adds (FADD2), spill traffic (STL / LDL) and
the register / shared-memory usage (cuobjdump -res-usage).

    python tools/sass_summary.py [lib.so] > profiles/sass_summary.json
"""
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

LIB = Path(sys.argv[1] if len(sys.argv) > 1 else
           Path(__file__).resolve().parents[1] / "paper_2007_06048_b200" / "libminimod_b200.so")
OPS = {"UTMALDG": r"\bUTMALDG", "LDS.128": r"\bLDS\.128\b", "STG.E.128": r"\bSTG\.E\.128\b",
       "FADD2": r"\bFADD2\b", "FFMA": r"\bFFMA\b", "FMUL": r"\bFMUL\b", "STL": r"\bSTL\b",
       "LDL": r"\bLDL\b", "BAR.SYNC": r"\bBAR\.SYNC", "SYNCS": r"\bSYNCS\."}


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:  # noqa: BLE001
        return name


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True,
                         text=True).stdout
    counts = defaultdict(lambda: defaultdict(int))
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        if cur is None or "/*" not in line:
            continue
        for k, pat in OPS.items():
            if re.search(pat, line):
                counts[cur][k] += 1
        counts[cur]["instructions"] += 1
    usage = {}
    fn = None
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", line)
        if fn and m:
            usage[fn] = {"registers": int(m.group(1)), "stack": int(m.group(2)),
                         "static_shared": int(m.group(3))}
    out = {}
    for fn, c in counts.items():
        d = demangle(fn)
        if not any(k in d for k in ("k_inner", "k_bnd", "k_p1", "k_cpml", "k_zslab", "k_vdv",
                                    "k_vdp", "k_epilogue")):
            continue
        out[d] = {**dict(c), **usage.get(fn, {})}
    print(json.dumps({"library": LIB.name, "arch": "sm_100a", "kernels": out}, indent=1,
                     sort_keys=True))


if __name__ == "__main__":
    main()
