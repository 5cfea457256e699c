"""GPU parity of the candidate logit head + CTR/CTCVR BCE against
the float64 oracle, alone and composed with the encoder stack (a trainable end-to-end loss)."""
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


def _labels(cfg, seg):
    L = seg.astype(np.int64).sum(1)
    return np.concatenate([synth.gen_user_labels(cfg, u, int(L[u])) for u in range(len(seg))] +
                          [np.zeros(0, np.uint8)])


def _oracle_head(seg, Z, lab, HP):
    h = oracle.build_jagged(seg)
    rows = oracle.candidate_rows(h["offsets"], h["n_static"], h["n_rt"], h["n_cand"])
    logits, loss, dzc, g = oracle.head_fwd_bwd(Z[rows], lab[rows], HP)
    dZ = np.zeros(Z.shape)
    dZ[rows] = dzc
    return logits, loss, dZ, g


@pytest.mark.parametrize("name", ["toy", "parity", "parity768"])
def test_head_parity(dev, name):
    cfg, seg, ts, X, _, _ = make_batch(name)
    dt = _dt(cfg)
    lab = _labels(cfg, seg)
    HP = synth.gen_head_params(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    hp = m.head_params_to_device(HP, dt, dev)
    z = torch.from_numpy(X).to(dev, dt)
    logits, loss, dz, g = m.head_fwd_bwd(jb, hp, z, torch.from_numpy(lab).to(dev))
    torch.cuda.synchronize()
    Lo, lo, dZo, go = _oracle_head(seg, z.float().cpu().numpy().astype(np.float64), lab, HP)
    tol = TOL[dt]
    errs = {"logits": rel_err(logits.cpu().numpy(), Lo), "loss": rel_err(loss.cpu().numpy(), lo),
            "dz": rel_err(dz.float().cpu().numpy(), dZo)}
    for k in go:
        errs["d" + k] = rel_err(g[k].cpu().numpy(), go[k])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (errs, bad)
    # non-candidate rows of dz are exactly zero
    h = oracle.build_jagged(seg)
    rows = oracle.candidate_rows(h["offsets"], h["n_static"], h["n_rt"], h["n_cand"])
    mask = np.ones(len(X), bool)
    mask[rows] = False
    assert not dz.float().cpu().numpy()[mask].any()


def test_head_deterministic_and_forward_only(dev):
    cfg, seg, ts, X, _, _ = make_batch("parity")
    lab = torch.from_numpy(_labels(cfg, seg)).to(dev)
    hp = m.head_params_to_device(synth.gen_head_params(cfg), torch.bfloat16, dev)
    jb = m.JaggedBatch.build(seg, ts, dev)
    z = torch.from_numpy(X).to(dev, torch.bfloat16)
    a = m.head_fwd_bwd(jb, hp, z, lab)
    b = m.head_fwd_bwd(jb, hp, z, lab)
    c = m.head_fwd_bwd(jb, hp, z, lab, want_grad=False)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    for k in a[3]:
        assert torch.equal(a[3][k], b[3][k]), k
    assert torch.equal(a[0], c[0]) and torch.equal(a[1], c[1]) and c[2] is None


def test_head_users_without_candidates(dev):
    seg = np.array([[2, 3, 1, 0], [1, 2, 0, 3], [0, 0, 0, 0], [4, 1, 2, 1]], np.int32)
    cfg, seg, ts, X, _, _ = make_batch("toy", seg=seg)
    lab = _labels(cfg, seg)
    HP = synth.gen_head_params(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    logits, loss, dz, g = m.head_fwd_bwd(jb, m.head_params_to_device(HP, torch.float32, dev),
                                         torch.from_numpy(X).to(dev), torch.from_numpy(lab).to(dev))
    Lo, lo, dZo, go = _oracle_head(seg, X.astype(np.float64), lab, HP)
    assert rel_err(logits.cpu().numpy(), Lo) <= 1e-4
    assert rel_err(loss.cpu().numpy(), lo) <= 1e-4
    assert rel_err(dz.cpu().numpy(), dZo) <= 1e-4


@pytest.mark.parametrize("name", ["toy", "parity"])
def test_stack_plus_head_end_to_end(dev, name):
    """Encoder (2 layers) + head: the loss and dX of the whole trainable path vs the oracle."""
    cfg, seg, ts, X, _, P = make_batch(name)
    dt = _dt(cfg)
    Ps = [P, synth.gen_layer_params(cfg, 1)]
    lab = _labels(cfg, seg)
    HP = synth.gen_head_params(cfg)
    jb = m.JaggedBatch.build(seg, ts, dev)
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    stack = m.HstuStack(lc, [m.params_to_device(p, dt, dev) for p in Ps], dt, dev)
    stack.bind(jb)
    z = stack.forward(torch.from_numpy(X).to(dev, dt))
    _, loss, dz, g = m.head_fwd_bwd(jb, m.head_params_to_device(HP, dt, dev), z, torch.from_numpy(lab).to(dev))
    dx = stack.backward(dz).float().cpu().numpy()
    torch.cuda.synchronize()
    # oracle: stack per user, head on the candidate rows, backward through the stack
    h = oracle.build_jagged(seg)
    ocfg = dict(d=cfg["d"], H=cfg["H"])
    Zo = np.zeros(X.shape)
    caches = []
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        zz, cc = oracle.stack_fwd_user(X[s:e], h["group_id"][s:e], int(h["n_static"][u]), int(h["n_rt"][u]),
                                       int(h["n_cand"][u]), ts[s:e], Ps, ocfg)
        Zo[s:e] = zz
        caches.append(cc)
    _, lo, dZo, go = _oracle_head(seg, Zo, lab, HP)
    dXo = np.zeros(X.shape)
    gW1 = [0.0, 0.0]
    for u in range(len(seg)):
        s, e = h["offsets"][u], h["offsets"][u + 1]
        dXo[s:e], gs = oracle.stack_bwd_user(dZo[s:e], caches[u], Ps, ocfg)
        for li in range(2):
            gW1[li] = gW1[li] + gs[li]["W1"]
    tol = TOL[dt]
    errs = {"loss": rel_err(loss.cpu().numpy(), lo), "dX": rel_err(dx, dXo),
            "dw_a": rel_err(g["w_a"].cpu().numpy(), go["w_a"])}
    for li in range(2):
        errs[f"L{li}.dW1"] = rel_err(stack.grads[li]["W1"].cpu().numpy(), gW1[li])
    assert all(v <= tol for v in errs.values()), errs
