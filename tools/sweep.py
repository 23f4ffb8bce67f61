"""Coarse/fine ratio and K sweep at 256^3 (BASELINE configs[4]) on W GPUs.

    python tools/sweep.py W out.jsonl [--handoff peer]
Runs bench.py under torchrun for N_t in {2^11, 2^12, 2^13, 2^14} (N_C = 2^9, the cfg3s
horizon: N_t / N_C = 4, 8, 16, 32 with cfg5's step sizes) and K in {1, 2, 3}, N_p = W,
and appends each JSON line to out.jsonl."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W, out = int(sys.argv[1]), sys.argv[2]
extra = sys.argv[3:]
port = 29600
for Nt in (2 ** 11, 2 ** 12, 2 ** 13, 2 ** 14):
    for K in (1, 2, 3):
        if K > W:
            continue
        port += 1
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
               "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.join(ROOT, "bench.py"), "--gpus", str(W), "--steps", "3", "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e", "--Nt", str(Nt), "--K", str(K), *extra]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
        if res.returncode != 0 or not lines:
            print(f"Nt={Nt} K={K}: failed\n{res.stdout[-2000:]}\n{res.stderr[-2000:]}", flush=True)
            continue
        d = json.loads(lines[-1])
        with open(out, "a") as f:
            f.write(lines[-1] + "\n")
        sp = d["speedup"]
        print(f"Nt={Nt} K={K}: ms={d['ms_per_step']:.0f} S={sp['S_measured']:.3f} "
              f"bound={sp['S_bound_eq_speedup_P229']:.3f} frac={sp['frac_of_bound']:.3f} "
              f"tc/tf={sp['tau_c_over_tau_f']:.3f} d={sp['defects']} "
              f"parity_ok={d.get('parity', {}).get('ok')}", flush=True)
