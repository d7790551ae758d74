"""Worker script for tests/test_cpu_host.py::test_launcher_runs_world2_gloo (not a test module):
each rank decodes its shard of requests with the CPU oracle and rank 0 writes the gathered map."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import torch.distributed as dist

    from oracle.llama_ref import RefLlama, greedy_ar
    from paper_2512_23858_b200.dist import env_rank, gather_generated, shard_requests
    from paper_2512_23858_b200.model import init_weights, preset

    out, n_req = sys.argv[1], int(sys.argv[2])
    rank, _, world = env_rank()
    dist.init_process_group("gloo")
    cfg = preset("tiny-target", n_layers=1)
    model = RefLlama(cfg, init_weights(cfg, 0, torch.float32))
    mine = {}
    for rid in shard_requests(n_req, world, rank):
        g = torch.Generator().manual_seed(1000 + rid)
        mine[rid] = greedy_ar(model, torch.randint(0, cfg.vocab, (8,), generator=g).tolist(), 4, 32)
    merged = gather_generated(mine, world)
    if rank == 0:
        Path(out).write_text(json.dumps({"world": world, "merged": {str(k): v for k, v in merged.items()}}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
