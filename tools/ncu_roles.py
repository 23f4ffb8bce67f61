"""Attribute ncu's warp-stall samples of a fused kernel to its warp roles and call sites.

    python tools/ncu_roles.py REPORT.ncu-rep LAUNCH LIB.so SOURCE.cuh [MANGLED_NAME]

REPORT: an `ncu --set full --import-source on` capture; LAUNCH: index of the launch in it;
LIB.so: the library that was profiled (same build); SOURCE.cuh: fused.cuh exactly as it was
built (e.g. `git show <rev>:paper_1409_8563_b200/csrc/fused.cuh > /tmp/f.cuh`).  The SASS
rows of ncu's source page are matched by offset to `nvdisasm -gi` of the library's cubin, whose
inline annotations give every instruction's call chain; each instruction is charged to the
outermost line inside producer_p / stage_a_p / stage_b_p.  Prints the share of all samples
per role and per call site, and how much of it is long-scoreboard (mbarrier wait) stall.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROLE_FUNCS = (("producer_p", "prod"), ("stage_a_p", "stageA"), ("stage_b_p", "stageB"))


def role_ranges(src_lines):
    starts = []
    for i, l in enumerate(src_lines, 1):
        for fn, name in ROLE_FUNCS:
            if re.match(r"__device__ __forceinline__ void %s\(" % fn, l):
                starts.append((i, name))
    starts.sort()
    out = []
    for k, (i, name) in enumerate(starts):
        end = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(src_lines)
        out.append((i, end, name))
    return out


def sass_chains(lib, mangled):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, check=True,
                       capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True,
                             text=True, check=True).stdout.split("\n")
    start = next(i for i, l in enumerate(txt) if l.startswith(".text." + mangled + ":"))
    info, cur, pending = {}, [], []
    for l in txt[start + 1:]:
        if l.startswith(".text.") or l.startswith(".section"):
            break
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
        if m:
            pending.append((os.path.basename(m.group(1)), int(m.group(2)),
                            m.group(3) and os.path.basename(m.group(3)), m.group(4) and int(m.group(4))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            if pending:
                cur, pending = pending, []
            info[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return info


def main():
    rep, launch, lib, src = sys.argv[1:5]
    src_lines = open(src).read().split("\n")
    ranges = role_ranges(src_lines)
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                           "--launch-skip", launch, "--launch-count", "1"],
                          capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    kname = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else "?"
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[k]
    data = [r for r in rows[k + 1:] if r and r[0].startswith("0x")]
    ix = {h: i for i, h in enumerate(hdr)}
    if len(sys.argv) > 5:
        mangled = sys.argv[5]
    else:  # fused_persist_kernel<KB, FusedCfgP<...>> of the product library, from ncu's name
        m = re.search(r"fused_persist_kernel<\(int\)(\d+), prk::FusedCfgP<([^>]*)>>", kname)
        if not m:
            sys.exit("pass the mangled kernel name for " + kname)
        args = "".join("Li%sE" % v for v in re.findall(r"\(int\)(-?\d+)", m.group(2)))
        mangled = ("_ZN3prk20fused_persist_kernelILi%sENS_9FusedCfgPI%sEEEEvNS_11StencilArgsENS_7TmaMapsE"
                   % (m.group(1), args))
    info = sass_chains(lib, mangled)

    def val(r, h):
        try:
            return float(r[ix[h]])
        except (ValueError, KeyError):
            return 0.0

    def role(chain):
        ls = []
        for fn, ln, fa, la in chain:
            if fn == os.path.basename(src):
                ls.append(ln)
            if fa == os.path.basename(src):
                ls.append(la)
        for ln in ls:
            for a, b, name in ranges:
                if a <= ln <= b:
                    return name, ln
        return "other", -1

    base = int(data[0][0], 16)
    tot = sum(val(r, "# Samples") for r in data)
    per_role, per_role_long, site = collections.Counter(), collections.Counter(), collections.Counter()
    mism = 0
    for r in data:
        chain, txt = info.get(int(r[0], 16) - base, ([], "?"))
        if txt.split()[:1] != r[1].strip().split()[:1]:
            mism += 1
        name, ln = role(chain)
        s, lsb = val(r, "# Samples"), val(r, "stall_long_sb")
        per_role[name] += s
        per_role_long[name] += lsb
        site[(name, ln)] += s
    print("# kernel:", kname)
    print("# %d SASS rows, %d opcode mismatches vs the library (must be 0), %d samples" % (len(data), mism, tot))
    print("# share of all warp-stall samples per role (long_sb = waiting on an mbarrier / global load)")
    for name, v in per_role.most_common():
        print("%-7s %5.1f %%   long_sb %5.1f %%" % (name, 100 * v / tot, 100 * per_role_long[name] / tot))
    print("# top call sites (outermost line inside the role function)")
    for (name, ln), v in site.most_common(16):
        text = src_lines[ln - 1].strip()[:100] if ln > 0 else ""
        print("%5.1f %%  %-7s l.%-4d %s" % (100 * v / tot, name, ln, text))


if __name__ == "__main__":
    main()
