"""GPU check of the whole training step (paper_2505_18654_b200.model.MTGRModel): sparse IDs ->
sharded dynamic-hash lookup -> Eq.4 tokens -> HSTU stack -> candidate head + BCE -> backward ->
sparse SGD, against the oracle composition (TableModel rows -> tokens_user -> stack -> head)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m
import synth
from tests.fixtures import make_batch, rel_err

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("name", ["toy", "parity"])
def test_full_training_step(dev, name, weighted):
    """weighted: the data-parallel form (R#20) with a global batch 3x this rank's users:
    every dense gradient (layers, head, token MLPs) comes out of the GradAggregator scaled by
    1/B_global and the sparse rows move by -lr/B_global x their summed gradients."""
    cfg, seg, ts, _, _, P = make_batch(name)
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
    d, e = cfg["d"], synth.EMB_DIM
    widths = synth.token_widths(cfg)
    Ps = [P, synth.gen_layer_params(cfg, 1)]
    TP, HP = synth.gen_token_params(cfg), synth.gen_head_params(cfg)
    ids = [synth.gen_user_feature_ids(cfg, u, seg[u]) for u in range(len(seg))]
    L = seg.astype(np.int64).sum(1)
    lab = np.concatenate([synth.gen_user_labels(cfg, u, int(L[u])) for u in range(len(seg))])
    user_ids = np.concatenate([i["u"].reshape(-1) for i in ids])
    item_ids = np.concatenate([np.concatenate([i[t].reshape(-1) for i in ids]) for t in "src"])
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(d, cfg["H"], cfg["groups"])
    lr = 0.05
    B_g = 3 * len(seg) if weighted else None
    wsc = 1.0 / B_g if weighted else 1.0
    model = m.MTGRModel(cfg, lc, Ps, TP, HP, widths, e, dt, dev, cap_user=4096, cap_item=1 << 16,
                        lr_sparse=lr, seed=3, n_users_global=B_g)
    model.bind(jb, seg)
    agg = None
    if weighted:
        from paper_2505_18654_b200.dp import GradAggregator
        agg = GradAggregator(B_g)
    loss, grads = model.step(torch.from_numpy(user_ids).to(dev), torch.from_numpy(item_ids).to(dev),
                             torch.from_numpy(lab).to(dev), now=1, aggregator=agg)
    torch.cuda.synchronize()
    # oracle: rows are the tables' init rows (rounded to the activation dtype on gather)
    rnd = (lambda a: a) if dt == torch.float32 else synth.round_bf16
    ut, it_ = oracle.TableModel(d, seed=3, scale=0.5), oracle.TableModel(e, seed=4, scale=0.5)
    h = oracle.build_jagged(seg)
    ocfg = dict(d=d, H=cfg["H"])
    Zo = np.zeros((int(L.sum()), d))
    st_c, tk_c, feats_u = [], [], []
    for u in range(len(seg)):
        s0, s1 = h["offsets"][u], h["offsets"][u + 1]
        f = {"u": rnd(ut.lookup(ids[u]["u"].reshape(-1)).astype(np.float32))}
        for t in "src":
            n_t = ids[u][t].shape[0]
            f[t] = rnd(it_.lookup(ids[u][t].reshape(-1)).astype(np.float32)).reshape(n_t, widths[t])
        feats_u.append(f)
        xo, tc = oracle.tokens_user(f, TP)
        zo, sc = oracle.stack_fwd_user(xo, h["group_id"][s0:s1], int(h["n_static"][u]), int(h["n_rt"][u]),
                                       int(h["n_cand"][u]), ts[s0:s1], Ps, ocfg)
        Zo[s0:s1] = zo
        st_c.append(sc); tk_c.append(tc)
    rows = oracle.candidate_rows(h["offsets"], h["n_static"], h["n_rt"], h["n_cand"])
    _, lo, dzc, go = oracle.head_fwd_bwd(Zo[rows], lab[rows], HP)
    dZo = np.zeros_like(Zo)
    dZo[rows] = dzc
    gW1, gtok = 0.0, 0.0
    dfe = []
    for u in range(len(seg)):
        s0, s1 = h["offsets"][u], h["offsets"][u + 1]
        dxo, gs = oracle.stack_bwd_user(dZo[s0:s1], st_c[u], Ps, ocfg)
        d_u, g_u = oracle.tokens_user_bwd(dxo, seg[u], tk_c[u], TP)
        gW1 = gW1 + gs[0]["W1"]
        gtok = gtok + g_u["s"]["w1"]
        dfe.append(d_u)
    tol = TOL[dt]
    errs = {"loss": rel_err(loss.cpu().numpy(), lo), "head.dw_a": rel_err(grads["head"]["w_a"].cpu().numpy(), wsc * go["w_a"]),
            "head.db_b": rel_err(grads["head"]["b_b"].cpu().numpy(), wsc * go["b_b"]),
            "L0.dW1": rel_err(grads["layers"][0]["W1"].cpu().numpy(), wsc * gW1),
            "tok.s.dw1": rel_err(grads["tokens"]["s"]["w1"].cpu().numpy(), wsc * gtok)}
    # sparse SGD: every item row moved by -lr * (sum of its occurrences' gradients)
    upd = {}
    for u in range(len(seg)):
        for t in "src":
            g = dfe[u][t].reshape(-1, e)
            for k, gr in zip(ids[u][t].reshape(-1).tolist(), g):
                upd[k] = upd.get(k, 0.0) + gr
    keys = np.array(sorted(upd)[:200], dtype=np.int64)
    slots = model.item_table.shard.find_or_insert(torch.from_numpy(keys).to(dev), insert=False)
    got = model.item_table.shard.gather(slots).cpu().numpy()
    ref = np.stack([oracle.init_row(4, int(k), e, 0.5) - lr * wsc * upd[int(k)] for k in keys])
    errs["item_rows"] = rel_err(got - np.stack([oracle.init_row(4, int(k), e, 0.5) for k in keys]),
                                ref - np.stack([oracle.init_row(4, int(k), e, 0.5) for k in keys]))
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (errs, bad)
