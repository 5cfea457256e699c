"""Worker of tests/test_gpu_embed.py::test_sharded_lookup_two_ranks (torchrun, NCCL): each rank
looks up its own skewed ID batch through the sharded table; the rows must equal the oracle's
single-table rows, and after one SGD step every rank must see the summed update."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2505_18654_b200 as m  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    rng = np.random.default_rng(100 + rank)
    ids = (rng.zipf(1.4, 20000) % 3000).astype(np.int64) * 131 + 7
    shard = m.HashEmbedding(dim=48, cap_v=16384, seed=21, init_scale=0.3, device=dev)
    emb = m.ShardedEmbedding(shard)
    rows, ctx = emb.lookup(torch.from_numpy(ids).to(dev), now=1)
    model = oracle.TableModel(48, seed=21, scale=0.3)
    np.testing.assert_array_equal(rows.cpu().numpy(), model.lookup(ids).astype(np.float32))
    # every rank's gradient = 1 per occurrence; the updated row of a key = init - lr * (#occurrences
    # over all ranks)
    g = torch.ones(len(ids), 48, device=dev)
    emb.backward_sgd(g, ctx, lr=0.01)
    all_ids = [None] * world
    dist.all_gather_object(all_ids, ids)
    cnt = {}
    for a in all_ids:
        for k in a.tolist():
            cnt[k] = cnt.get(k, 0) + 1
    rows2, _ = emb.lookup(torch.from_numpy(ids).to(dev), now=2)
    ref = np.stack([oracle.init_row(21, int(k), 48, 0.3) - 0.01 * cnt[int(k)] for k in ids])
    np.testing.assert_allclose(rows2.cpu().numpy(), ref, rtol=0, atol=1e-4)
    dist.barrier()
    if rank == 0:
        print("EMBED_DIST_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
