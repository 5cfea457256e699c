"""GPU parity of the Eq.4 token construction against the float64
oracle, and of the whole trainable path: features -> tokens -> encoder stack -> candidate head
-> BCE, backward to the feature embeddings and every parameter."""
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


def _dt(cfg):
    return torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16


def _features(cfg, seg):
    per_user = [synth.gen_user_features(cfg, u, seg[u]) for u in range(len(seg))]
    k = synth.token_widths(cfg)
    packed = {t: np.concatenate([f[t] for f in per_user] + [np.zeros((0, k[t]), np.float32)])
              for t in synth.TOKEN_TYPES}
    return per_user, packed


def _embed(cfg, seg, ts, dev, TP, packed):
    dt = _dt(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    emb = m.TokenEmbed(cfg["d"], synth.token_widths(cfg), m.TokenEmbed.params_to_device(TP, dt, dev), dt, dev)
    emb.bind(jb, seg)
    feats = {t: torch.from_numpy(v).to(dev, dt) for t, v in packed.items()}
    return jb, emb, feats


@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_token_construction_parity(dev, name):
    cfg, seg, ts, _, dZ, _ = make_batch(name)
    dt = _dt(cfg)
    per_user, packed = _features(cfg, seg)
    TP = synth.gen_token_params(cfg)
    jb, emb, feats = _embed(cfg, seg, ts, dev, TP, packed)
    x = emb.forward(feats)
    dfe, g = emb.backward(torch.from_numpy(dZ).to(dev, dt))
    torch.cuda.synchronize()
    h = oracle.build_jagged(seg)
    Xo = np.zeros((len(dZ), cfg["d"]))
    dfo = {t: [] for t in synth.TOKEN_TYPES}
    go = None
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        Xo[s:e], caches = oracle.tokens_user(per_user[u], TP)
        d_u, g_u = oracle.tokens_user_bwd(dZ[s:e], seg[u], caches, TP)
        for t in dfo:
            dfo[t].append(d_u[t])
        go = g_u if go is None else {t: {k: go[t][k] + g_u[t][k] for k in go[t]} for t in go}
    tol = TOL[dt]
    errs = {"X": rel_err(x.float().cpu().numpy(), Xo)}
    for t in synth.TOKEN_TYPES:
        errs["dfeat_" + t] = rel_err(dfe[t].float().cpu().numpy(), np.concatenate(dfo[t]))
    for t in ("s", "r", "c"):
        for k in go[t]:
            errs[f"{t}.d{k}"] = rel_err(g[t][k].cpu().numpy(), go[t][k])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (errs, bad)


def test_token_empty_types(dev):
    """Users without S / R / candidate tokens, and an empty user."""
    seg = np.array([[2, 0, 3, 0], [1, 4, 0, 2], [0, 0, 0, 0], [3, 2, 1, 1]], np.int32)
    cfg, seg, ts, _, dZ, _ = make_batch("toy", seg=seg)
    per_user, packed = _features(cfg, seg)
    TP = synth.gen_token_params(cfg)
    jb, emb, feats = _embed(cfg, seg, ts, dev, TP, packed)
    x = emb.forward(feats).cpu().numpy()
    h = oracle.build_jagged(seg)
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        assert rel_err(x[s:e], oracle.tokens_user(per_user[u], TP)[0]) <= 1e-4


@pytest.mark.parametrize("name", ["toy", "parity"])
def test_full_trainable_path(dev, name):
    """features -> tokens (Eq.4) -> 2-layer encoder -> candidate head -> BCE; backward to the
    feature embeddings; loss and feature / token-MLP gradients vs the oracle composition."""
    cfg, seg, ts, _, _, P = make_batch(name)
    dt = _dt(cfg)
    Ps = [P, synth.gen_layer_params(cfg, 1)]
    per_user, packed = _features(cfg, seg)
    TP, HP = synth.gen_token_params(cfg), synth.gen_head_params(cfg)
    L = seg.astype(np.int64).sum(1)
    lab = np.concatenate([synth.gen_user_labels(cfg, u, int(L[u])) for u in range(len(seg))])
    jb, emb, feats = _embed(cfg, seg, ts, dev, TP, packed)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    stack = m.HstuStack(lc, [m.params_to_device(p, dt, dev) for p in Ps], dt, dev)
    stack.bind(jb)
    x = emb.forward(feats)
    z = stack.forward(x.contiguous())
    _, loss, dz, _ = m.head_fwd_bwd(jb, m.head_params_to_device(HP, dt, dev), z, torch.from_numpy(lab).to(dev))
    dx = stack.backward(dz)
    dfe, g = emb.backward(dx)
    torch.cuda.synchronize()
    # oracle composition
    h = oracle.build_jagged(seg)
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    T = int(L.sum())
    Zo = np.zeros((T, cfg["d"]))
    st_c, tk_c = [], []
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        xo, tc = oracle.tokens_user(per_user[u], TP)
        zo, sc = oracle.stack_fwd_user(xo, h["group_id"][s:e], int(h["n_static"][u]), int(h["n_rt"][u]),
                                       int(h["n_cand"][u]), ts[s:e], Ps, ocfg)
        Zo[s:e] = zo
        st_c.append(sc)
        tk_c.append(tc)
    rows = oracle.candidate_rows(h["offsets"], h["n_static"], h["n_rt"], h["n_cand"])
    _, lo, dzc, _ = oracle.head_fwd_bwd(Zo[rows], lab[rows], HP)
    dZo = np.zeros_like(Zo)
    dZo[rows] = dzc
    dfo = {t: [] for t in synth.TOKEN_TYPES}
    gs = None
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        dxo, _ = oracle.stack_bwd_user(dZo[s:e], st_c[u], Ps, ocfg)
        d_u, g_u = oracle.tokens_user_bwd(dxo, seg[u], tk_c[u], TP)
        for t in dfo:
            dfo[t].append(d_u[t])
        gs = g_u if gs is None else {t: {k: gs[t][k] + g_u[t][k] for k in gs[t]} for t in gs}
    tol = TOL[dt]
    errs = {"loss": rel_err(loss.cpu().numpy(), lo)}
    for t in synth.TOKEN_TYPES:
        errs["dfeat_" + t] = rel_err(dfe[t].float().cpu().numpy(), np.concatenate(dfo[t]))
    for t in ("s", "c"):
        errs[f"{t}.dw1"] = rel_err(g[t]["w1"].cpu().numpy(), gs[t]["w1"])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (errs, bad)
