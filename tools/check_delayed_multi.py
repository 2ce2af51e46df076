"""f1 across ranks (run under torchrun, NCCL): the delayed, pipelined refresh with owner-sharded roots -- each rank's
chunks on its own lowest-priority stream, the rank-uniform all-gather step -- must adopt, at every kappa boundary,
roots bit-identical to a synchronous single-GPU refresh of the same statistics snapshot.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
        tools/check_delayed_multi.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2002_09018_b200 as shp  # noqa: E402
import synth  # noqa: E402
from paper_2002_09018_b200.schedule import DelayedRefresh  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    # unequal owned counts across ranks: mixed sizes, some one-sided
    shapes = [(1024, 1024), (512, 2048), (300, 200), (128, 128), (2048, 640), (40, 700), (1024, 512)]
    plan = shp.make_plan(shapes, 512, 1024, world)
    plan1 = shp.make_plan(shapes, 512, 1024, 1)
    Gs = [torch.zeros(s, dtype=torch.float32, device=dev) for s in shapes]
    table = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
    table1 = shp.TensorTable(Gs, [torch.zeros_like(G) for G in Gs])
    stats = torch.zeros(plan.stats_elems, dtype=torch.float32, device=dev)
    stats1 = torch.zeros(plan1.stats_elems, dtype=torch.float32, device=dev)
    kappa = 4
    dr = DelayedRefresh(plan, stats, torch.zeros_like(stats), rank, world, kappa=kappa, spread=3, fp64_iters="auto")
    counts = [sum(int(g["count"]) for g in plan.groups_of(r)) for r in range(world)]
    snaps, bad, adopted = {}, 0, 0
    for t in range(3 * kappa + 1):
        for i, (G, s) in enumerate(zip(Gs, shapes)):
            G.copy_(torch.from_numpy(synth.gaussian(s, 1000 * t + i)))
        shp.stats_update(table, plan, stats, 1.0, 1.0, rank)
        shp.stats_update(table1, plan1, stats1, 1.0, 1.0, -1)
        if t % kappa == 0:
            snaps[t] = stats1.clone()
        if dr.step(t):
            adopted += 1
            ref = torch.zeros_like(stats1)
            shp.refresh_group_roots(plan1, snaps[t - kappa], ref, 0, fp64_iters="auto")
            torch.cuda.synchronize()
            for b, b1 in zip(plan.blocks, plan1.blocks):
                for side in ("left", "right"):
                    if b[f"p_{side}"]:
                        n = int(b["rows"] if side == "left" else b["cols"])
                        ld = int(b[f"{side}_ld"])
                        o, o1 = int(b[f"{side}_off"]), int(b1[f"{side}_off"])
                        if not torch.equal(dr.current[o:o + n * ld], ref[o1:o1 + n * ld]):
                            bad += 1
    torch.cuda.synchronize()
    t_ = torch.tensor([bad, adopted], device=dev)
    dist.all_reduce(t_)
    if rank == 0:
        print(f"world {world}: owned roots per rank {counts}, chunk {dr.chunk}, chunk steps {dr.n_steps}, "
              f"adoptions {int(t_[1].item()) // world}, roots differing from the synchronous 1-GPU refresh "
              f"(summed over ranks and adoptions) = {int(t_[0].item())}", flush=True)
    dist.destroy_process_group()
    if int(t_[0].item()) != 0 or int(t_[1].item()) != 3 * world:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
