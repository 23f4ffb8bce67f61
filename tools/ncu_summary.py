"""Summarise an ncu --set full report: one line per kernel launch."""
import csv
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB_r"), ("dram__bytes_write.sum", "MB_w"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__t_bytes.sum", "L2_MB"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_shared_mem", "occ_smem"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank_conf")]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "mio_throttle", "lg_throttle",
          "math_pipe_throttle", "selected", "not_selected", "no_instruction", "drain", "branch_resolving"]


SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def main(rep):
    hdr, units, data = rows(rep)
    for r in data:
        name = r[hdr.index("Kernel Name")]
        parts = [name[:40]]
        for m, short in WANT:
            if m in hdr:
                i = hdr.index(m)
                v = r[i]
                if units[i] in SCALE:  # byte counters reported in MB whatever ncu's unit
                    v = f"{float(v.replace(',', '')) * SCALE[units[i]]:.3f}"
                parts.append(f"{short}={v}")
        st = []
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in hdr:
                st.append(f"{s}={float(r[hdr.index(m)]):.2f}")
        print(" ".join(parts))
        print("   stalls/issue: " + " ".join(st))


if __name__ == "__main__":
    main(sys.argv[1])
