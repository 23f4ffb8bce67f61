"""Turn gpurun_out ncu outputs into the committed profiles/ summaries.

    python tools/make_profiles.py <round> <launches.csv> <full.ncu-rep> [n] [tag]
Writes profiles/r<round>_launch_shares_cfg3p.txt, r<round>_launches_cfg3p.csv,
r<round>_ncu_full_k<n>_summary.txt and updates profiles/ncu_summary.json
(dram bytes per RK4 step for the fused and four-stage paths)."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 256
tag = sys.argv[5] + "_" if len(sys.argv) > 5 else ""
P = os.path.join(ROOT, "profiles")

rows = list(csv.reader(open(launches)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot, cnt = collections.Counter(), collections.Counter()
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    tot[d["Kernel Name"]] += v
    cnt[d["Kernel Name"]] += 1
T = sum(tot.values())
with open(os.path.join(P, f"r{rnd}_launch_shares_cfg3p.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    f.write("# command: python bench.py --config cfg3p --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
            "  (256^3, cfg3's dt/Dt; N_p=1, K=1)\n")
    f.write("# every launch of the run: serial fine reference, coarse timing, 3 warm-up + 1 timed Parareal"
            " solve, four-stage comparison timing\n")
    for k, v in tot.most_common():
        f.write(f"{k[:78]:78s} launches={cnt[k]:6d} total_us={v / 1e3:10.1f} share={100 * v / T:6.2f}%"
                f" mean_ns={v / cnt[k]:.0f}\n")
with open(os.path.join(P, f"r{rnd}_launches_cfg3p.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "gpu__time_duration_ns"])
    for d in data:
        w.writerow([d["ID"], d["Kernel Name"], d["Grid Size"], d["Block Size"], d["Metric Value"]])

out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                     capture_output=True, text=True).stdout
open(os.path.join(P, f"r{rnd}_ncu_full_{tag}k{n}_summary.txt"), "w").write(out)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
scale = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1}
per = collections.defaultdict(list)
for row in r[2:]:
    b = sum(float(row[h.index(m)]) * scale[units[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    per[row[h.index("Kernel Name")]].append((b, float(row[h.index("gpu__time_duration.sum")])))
avg = {k: [sum(x[0] for x in v) / len(v), sum(x[1] for x in v) / len(v)] for k, v in per.items()}
fused = sum(b for k, (b, t) in avg.items() if "fused_" in k)
four = sum(b for k, (b, t) in avg.items() if any(f"stencil_kernel<{i}," in k for i in (1, 2, 3, 4)))
p = os.path.join(P, "ncu_summary.json")
js = json.load(open(p)) if os.path.exists(p) else {}
js.setdefault("fine_step_dram_bytes", {})
js.setdefault("fine_step_algorithmic_bytes", {})
if fused:
    js["fine_step_dram_bytes"].setdefault("fused", {})[str(n)] = fused
    js["fine_step_algorithmic_bytes"].setdefault("fused", {})[str(n)] = 56 * n ** 3
if four:
    js["fine_step_dram_bytes"].setdefault("four_stage", {})[str(n)] = four
    js["fine_step_algorithmic_bytes"].setdefault("four_stage", {})[str(n)] = 128 * n ** 3
js.setdefault("per_launch_bytes_and_us", {}).update(avg)
js["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) and gpu__time_duration (us) "
              f"from ncu --set full --clock-control none, round {rnd}, tools/profile_kernels.py {n}")
json.dump(js, open(p, "w"), indent=1)
print(out)
print("fused", fused, "four", four)
