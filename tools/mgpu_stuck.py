"""NCCL hand-off failure path (run under torchrun with 2 ranks, 2 GPUs).

Rank 0 never calls pr_parareal (a stuck predecessor); rank 1 calls it with
PR_NCCL_TIMEOUT_S=5 and must get PR_ENCCL naming its rank and iteration
(SURVEY 8(b) error conventions).  Prints one JSON line on rank 1."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1409_8563_b200 as pr  # noqa: E402


def main():
    os.environ["PR_NCCL_TIMEOUT_S"] = "5"
    handoff = sys.argv[1] if len(sys.argv) > 1 else "nccl"
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    n = 32
    g = pr.Grid(pr.Problem(n), local)
    pr.comm_init_torch(g)
    u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(g, u0)
    ok = True
    if rank == 1:
        flags = pr.PR_FLAG_PEER_HANDOFF if handoff == "peer" else 0
        info = {"handoff": handoff}
        try:
            pr.pr_parareal(g, pr.PararealCfg(2, 4, 16, 2, flags=flags), u0, torch.empty_like(u0), None)
            info["error"] = None
            ok = False
        except pr.PrError as e:
            info.update(status=e.status, error=str(e))
            ok = e.status == 4 and "rank 1, iteration" in str(e)
        info["ok"] = ok
        print(json.dumps(info), flush=True)
    dist.barrier()
    os._exit(0 if ok else 1)  # rank 1's communicator was aborted: skip teardown


if __name__ == "__main__":
    main()
