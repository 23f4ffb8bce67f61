"""Static SASS instruction mix of the library's persistent kernels (evidence of the
Blackwell paths: UTMALDG = TMA tensor loads, LDGSTS = cp.async, SYNCS = mbarrier,
LDTM / STTM = tcgen05.ld / tcgen05.st tensor-memory moves, UTCATOMSWS = tcgen05.alloc).

    python tools/sass_mix.py [lib.so]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTMALDG", "LDGSTS", "SYNCS", "LDTM", "STTM", "UTCATOMSWS", "DFMA", "DMUL", "DADD", "LDS",
        "STS", "STG", "BAR"]


def mix(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, counts = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            counts[cur][m.group(2)] += 1
    return counts


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1409_8563_b200", "libparareal.so")
    for f, c in mix(lib).items():
        if any(k in f for k in ("fused", "comb", "onestep", "coarse_persist", "z2")):
            dem = subprocess.run(["c++filt"], input=f, capture_output=True, text=True).stdout.strip()
            print(dem[:150])
            print("   " + "  ".join(f"{k}={c[k]}" for k in KEYS if c[k]))


if __name__ == "__main__":
    main()
