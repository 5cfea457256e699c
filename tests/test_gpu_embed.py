"""GPU checks of the dynamic hash embedding and the sharded lookup
against the oracle's semantics.  Slot numbers / bucket positions / unique order are
implementation choices: compared are the rows (bit-exact init, SGD within fp32 summation
order), the key -> slot function (consistent, injective), the unique set and the inverse map."""
import os
import subprocess
import sys

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


def _ids(seed, n, vocab):
    rng = np.random.default_rng(seed)
    # Zipf-like skew: many repeats of hot ids, plus negative / huge ids
    ids = (rng.zipf(1.3, n) % vocab).astype(np.int64) * 7919 - vocab
    ids[::97] = rng.integers(-(1 << 62), 1 << 62, len(ids[::97]))
    return ids


def test_find_or_insert_and_init_rows(dev):
    ids = _ids(0, 20000, 5000)
    t = m.HashEmbedding(dim=40, cap_v=8192, seed=11, init_scale=0.25, device=dev)
    slots = t.find_or_insert(torch.from_numpy(ids).to(dev), now=1).cpu().numpy()
    u = np.unique(ids)
    # consistent and injective key -> slot
    mp = {}
    for k, s in zip(ids.tolist(), slots.tolist()):
        assert s >= 0
        assert mp.setdefault(k, s) == s
    assert len(set(mp.values())) == len(u)
    assert t.stats()["fresh_slots"] == len(u) and t.stats()["failed"] == 0
    # rows bit-exact vs the shared counter-based generator
    rows = t.gather(torch.from_numpy(slots).to(dev)).cpu().numpy()
    for i in range(0, len(ids), 211):
        np.testing.assert_array_equal(rows[i], oracle.init_row(11, int(ids[i]), 40, 0.25))
    # lookup without insert finds every key, misses unknown ones
    s2 = t.find_or_insert(torch.from_numpy(u).to(dev), insert=False).cpu().numpy()
    assert all(mp[k] == s for k, s in zip(u.tolist(), s2.tolist()))
    miss = t.find_or_insert(torch.tensor([123456789123], device=dev), insert=False).cpu().numpy()
    assert miss[0] == -1


def test_capacity_failure_is_reported(dev):
    t = m.HashEmbedding(dim=8, cap_v=100, cap_k=256, device=dev)
    s = t.find_or_insert(torch.arange(150, device=dev, dtype=torch.int64)).cpu().numpy()
    assert (s >= 0).sum() == 100 and (s == -2).sum() == 50 and t.stats()["failed"] == 50


def test_sgd_evict_expand(dev):
    ids = _ids(1, 5000, 800)
    model = oracle.TableModel(16, seed=5, scale=0.1)
    t = m.HashEmbedding(dim=16, cap_v=4096, seed=5, init_scale=0.1, device=dev)
    ti = torch.from_numpy(ids).to(dev)
    slots = t.find_or_insert(ti, now=100)
    model.lookup(ids, now=100)
    g = np.random.default_rng(2).standard_normal((len(ids), 16)).astype(np.float32)
    t.sgd(slots, torch.from_numpy(g).to(dev), lr=0.01)
    model.sgd(ids, g, 0.01)
    got = t.gather(slots).cpu().numpy()
    ref = model.lookup(ids, now=100)
    _, inv, cnt = np.unique(ids, return_inverse=True, return_counts=True)
    absum = np.zeros((len(cnt), 16))
    np.add.at(absum, inv, np.abs(g))
    bound = 0.01 * (cnt[:, None] * 2.0 ** -23) * absum + 1e-6  # fp32 atomics in any order
    assert (np.abs(got - ref) <= bound[inv]).all()
    # touch half of the keys later, evict the rest
    u = np.unique(ids)
    late = u[::2]
    t.find_or_insert(torch.from_numpy(late).to(dev), now=200)
    model.lookup(late, now=200)
    t.evict(ts_before=150)
    model.evict(150)
    present = t.find_or_insert(torch.from_numpy(u).to(dev), insert=False).cpu().numpy()
    assert ((present >= 0) == np.isin(u, late)).all()
    assert t.stats()["free_stack"] == len(u) - len(late)
    # re-insert an evicted key: fresh init row, recycled slot
    k = int(u[1])
    s = t.find_or_insert(torch.tensor([k], device=dev), now=300)
    np.testing.assert_array_equal(t.gather(s).cpu().numpy()[0], oracle.init_row(5, k, 16, 0.1))
    assert t.stats()["free_stack"] == len(u) - len(late) - 1
    # expand the key structure only: same slots, same rows
    before = t.find_or_insert(torch.from_numpy(late).to(dev), insert=False)
    rows_before = t.gather(before).cpu().numpy()
    t.expand(4 * t.cap_k)
    after = t.find_or_insert(torch.from_numpy(late).to(dev), insert=False)
    assert torch.equal(before, after)
    np.testing.assert_array_equal(t.gather(after).cpu().numpy(), rows_before)


def test_unique_and_segment_sum(dev):
    ids = _ids(3, 30000, 3000)
    u, inv = m.unique(torch.from_numpy(ids).to(dev))
    u, inv = u.cpu().numpy(), inv.cpu().numpy()
    np.testing.assert_array_equal(np.sort(u), np.unique(ids))
    np.testing.assert_array_equal(u[inv], ids)
    g = torch.randn(len(ids), 24, device=dev)
    s = m.segment_sum(g, torch.from_numpy(inv).to(dev), len(u)).cpu().numpy()
    ref = np.zeros((len(u), 24))
    np.add.at(ref, inv, g.cpu().numpy().astype(np.float64))
    np.testing.assert_allclose(s, ref, rtol=1e-5, atol=1e-4)


def test_sharded_lookup_single_rank(dev):
    ids = _ids(4, 12000, 2000)
    shard = m.HashEmbedding(dim=32, cap_v=8192, seed=9, init_scale=0.2, device=dev)
    emb = m.ShardedEmbedding(shard)
    rows, ctx = emb.lookup(torch.from_numpy(ids).to(dev), now=1)
    model = oracle.TableModel(32, seed=9, scale=0.2)
    np.testing.assert_array_equal(rows.cpu().numpy(), model.lookup(ids).astype(np.float32))
    g = torch.randn(len(ids), 32, device=dev)
    emb.backward_sgd(g, ctx, lr=0.05)
    gn = g.cpu().numpy()
    model.sgd(ids, gn, 0.05)
    rows2, _ = emb.lookup(torch.from_numpy(ids).to(dev), now=2)
    # fp32 sums of n occurrences in an unspecified order: |error| <= lr * n * 2^-23 * sum|g| per
    # column (the standard recursive-summation bound), plus the rounding of the row itself
    _, inv, cnt = np.unique(ids, return_inverse=True, return_counts=True)
    absum = np.zeros((len(cnt), 32))
    np.add.at(absum, inv, np.abs(gn))
    bound = 0.05 * (cnt[:, None] * 2.0 ** -23) * absum + 1e-6
    err = np.abs(rows2.cpu().numpy() - model.lookup(ids))
    assert (err <= bound[inv]).all(), float((err / bound[inv]).max())


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_sharded_lookup_two_ranks():
    """2 ranks over NCCL: rows identical to the single-table oracle; updates land on the owner."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tools", "embed_dist_check.py")]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "EMBED_DIST_OK" in r.stdout
