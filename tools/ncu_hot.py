"""Top SASS lines by warp-stall samples for one kernel of an ncu report."""
import csv, subprocess, sys
rep, which = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(which), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
which = 0
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]; blocks.append(cur); continue
    if cur and len(r) > 5 and r[0].startswith("0x"):
        cur[1].append((int(r[2]), int(r[5]), r[1].strip(), r[0]))
name, lines = blocks[which]
tot = sum(l[0] for l in lines)
print(name, "samples", tot)
for s, ex, src, addr in sorted(lines, reverse=True)[:top]:
    print(f"{s:6d} {100*s/tot:5.1f}% ex={ex:9d} {addr[-5:]} {src}")
