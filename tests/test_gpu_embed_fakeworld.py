"""Distributed embedding lookup of P:355 (two-stage ID unique + all-to-all) with W = 2 and 4
shards on ONE GPU: every shard is its own HashEmbedding / ShardedEmbedding, driven by its own
host thread (one "rank" each), and only the all-to-all is emulated, by a buffer exchange between
the threads (split, hand over, concatenate in source-rank order: the semantics of
torch.distributed.all_to_all_single).  Every other step — stage-1 unique, owner partition,
stage-2 unique, find-or-insert + gather on the owner, the row moves back, the backward segment
sums and the owner SGD — runs in libmtgr exactly as with NCCL.  Checked against the oracle's
single-table model: looked-up rows bit-exact, rows after one summed update within the fp32
summation-order bound."""
import threading

import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


class _Hub:
    def __init__(self, W):
        self.W = W
        self.bar = threading.Barrier(W)
        self.slots = [None] * W


class _FakeDist:
    """The two collectives ShardedEmbedding uses, over threads of one process."""

    def __init__(self, rank, hub):
        self.rank, self.hub = rank, hub

    def get_world_size(self, group=None):
        return self.hub.W

    def all_to_all_single(self, out, inp, output_split_sizes=None, input_split_sizes=None, group=None):
        W = self.hub.W
        sizes = input_split_sizes or [inp.shape[0] // W] * W
        torch.cuda.synchronize()
        self.hub.slots[self.rank] = [p.clone() for p in torch.split(inp, sizes)]
        torch.cuda.synchronize()
        self.hub.bar.wait()
        got = torch.cat([self.hub.slots[src][self.rank] for src in range(W)])
        assert got.shape[0] == out.shape[0]
        out.copy_(got)
        torch.cuda.synchronize()
        self.hub.bar.wait()


def _ids(seed, n, vocab):
    rng = np.random.default_rng(seed)
    ids = (rng.zipf(1.2, n) % vocab).astype(np.int64) * 104729 + 17
    ids[::89] = rng.integers(-(1 << 60), 1 << 60, len(ids[::89]))
    return ids


@pytest.mark.parametrize("W", [2, 4])
def test_sharded_lookup_fake_world(dev, W):
    dim, seed, scale, lr = 16, 21, 0.3, 0.07
    ids = [_ids(100 + r, 6000 + 1500 * r, 2500) for r in range(W)]  # ragged per-rank batches
    grads = [np.random.default_rng(200 + r).standard_normal((len(ids[r]), dim)).astype(np.float32)
             for r in range(W)]
    hub = _Hub(W)
    out = [dict() for _ in range(W)]
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(dev)
            emb = m.ShardedEmbedding(m.HashEmbedding(dim=dim, cap_v=1 << 14, seed=seed, init_scale=scale, device=dev))
            emb.world, emb.dist = W, _FakeDist(r, hub)
            x = torch.from_numpy(ids[r]).to(dev)
            rows, ctx = emb.lookup(x, now=1)
            out[r]["rows"] = rows.cpu().numpy()
            out[r]["owned"] = int(ctx["slots"].numel())
            emb.backward_sgd(torch.from_numpy(grads[r]).to(dev), ctx, lr)
            rows2, _ = emb.lookup(x, now=2)
            out[r]["rows2"] = rows2.cpu().numpy()
        except Exception as e:  # surfaced on the main thread
            errs.append(e)
            hub.bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    model = oracle.TableModel(dim, seed=seed, scale=scale)
    for r in range(W):  # first lookup: the tables' init rows, whoever owns them
        np.testing.assert_array_equal(out[r]["rows"], model.lookup(ids[r]).astype(np.float32))
    # every distinct id is owned by exactly one shard
    assert sum(o["owned"] for o in out) == len(np.unique(np.concatenate(ids)))
    allid, allg = np.concatenate(ids), np.concatenate(grads)
    model.sgd(allid, allg, lr)
    _, inv, cnt = np.unique(allid, return_inverse=True, return_counts=True)
    absum = np.zeros((len(cnt), dim))
    np.add.at(absum, inv, np.abs(allg))
    bound_all = lr * (cnt[:, None] * 2.0 ** -23) * absum + 1e-6
    uid = np.unique(allid)
    for r in range(W):
        ref = model.lookup(ids[r], now=2)
        b = bound_all[np.searchsorted(uid, ids[r])]
        err = np.abs(out[r]["rows2"] - ref)
        assert (err <= b).all(), (r, float((err / b).max()))
