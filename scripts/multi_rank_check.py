"""N ranks (torchrun) each track their block-cyclic shard of a range with libpp200 on their GPU
(ranks share GPUs round-robin when there are fewer GPUs than ranks, over gloo), rank 0 gathers
the records with paper_1505_00383_b200.shard.distributed_track_all and writes them to OUT.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        scripts/multi_rank_check.py SYSTEM PREC LO HI BLOCK OUT.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    system, prec, lo, hi, block, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
    import torch
    import torch.distributed as dist

    import paper_1505_00383_b200 as P
    from paper_1505_00383_b200.shard import FIELDS, distributed_track_all

    world = int(os.environ["WORLD_SIZE"])
    ndev = torch.cuda.device_count()
    device = int(os.environ.get("LOCAL_RANK", "0")) % max(1, ndev)
    dist.init_process_group("nccl" if ndev >= world else "gloo")
    f = P.parse_system(open(os.path.join(ROOT, "tests", "data", f"{system}.sys")).read())
    g, st = P.total_degree_start(f, prec)
    h = P.make_homotopy(f, g, P.random_gamma(1), prec)

    def fn(a, b, shard):
        sol = P.track_all(h, st, lo=a, hi=b, device=device, shard=shard)
        return {k: getattr(sol, k) for k in FIELDS}

    merged = distributed_track_all(fn, lo, hi, dist, block=block)
    if dist.get_rank() == 0:
        np.savez(out, **merged)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
