"""Config-4 time steps on N GPUs with parallel.ShardedTimeLoop (K5 regions
split over the ranks with the loads all-reduced, the theta-step solve on
z-slabs with NCCL halo / partial-sum exchange). Launch:

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port 29600 tools/sharded_run.py [cfg] [steps]

Rank 0 prints one JSON line: device ms per step (CUDA events around
tg_sim_advance on each rank's stream, max over ranks) and CG iterations."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2511_20432_b200 as tg
    from paper_2511_20432_b200 import parallel
    cfg = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "cfg4_large.cfg")
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl")
    d = parallel.Dist(dist.get_rank(), dist.get_world_size(), f"cuda:{local}")
    sim = tg.Simulation(cfg, device=local)
    loop = parallel.ShardedTimeLoop(sim, d)
    loop.reset()
    loop.step()  # warm-up
    ctx = sim.context()
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    its, _ = loop.step(steps)
    prof = ctx.profile()
    ms = torch.tensor([prof["step_ms"] / steps], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if d.rank == 0:
        print(json.dumps({"workload": os.path.basename(cfg), "n_gpus": d.world,
                          "ms_per_step": float(ms.item()), "steps": steps,
                          "cg_iterations_per_step": its / steps}), flush=True)
    sim.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
