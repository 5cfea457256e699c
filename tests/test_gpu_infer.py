"""Inference fast path: the CUDA-graph-captured forward of `InferenceSession`
against the float64 oracle, on requests shaped like the `infer` config (d=768, 3 heads,
candidates sharing the user prefix) but short enough for the oracle."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_18654_b200 as m
import synth
from paper_2505_18654_b200.infer import InferenceSession
from tests.fixtures import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _request(cfg, seg, x_stream=0):
    L = seg.astype(np.int64).sum(1)
    ts = np.concatenate([synth.gen_user_ts(cfg, u, seg[u]) for u in range(len(seg))])
    X = np.concatenate([synth.gen_user_x(cfg, u + 1000 * x_stream, int(L[u])) for u in range(len(seg))])
    return ts, X


def _oracle(cfg, seg, ts, X, Ps):
    out = []
    off = np.concatenate([[0], np.cumsum(seg.astype(np.int64).sum(1))])
    for u in range(len(seg)):
        a, b = int(off[u]), int(off[u + 1])
        gid = oracle.build_jagged(seg[u:u + 1])["group_id"]
        nU, nS, nR, K = (int(v) for v in seg[u])
        z, _ = oracle.stack_fwd_user(X[a:b], gid, nU + nS, nR, K, ts[a:b], Ps, dict(d=cfg["d"], H=cfg["H"]))
        out.append(z)
    return np.concatenate(out)


def test_graph_forward_matches_oracle_and_replays(dev):
    cfg = synth.config("infer", n_layers=2)
    seg = np.array([[32, 420, 60, 50], [32, 180, 0, 70], [32, 300, 100, 125]], dtype=np.int32)
    Ps = [synth.gen_layer_params(cfg, li) for li in range(cfg["n_layers"])]
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    ts, X = _request(cfg, seg)
    sess = InferenceSession(lc, [m.params_to_device(P, torch.bfloat16, dev) for P in Ps],
                            torch.bfloat16, dev, seg, ts)
    sess.set_request(torch.from_numpy(X).to(dev, torch.bfloat16))
    sess.capture()
    z = sess.run().float().cpu().numpy()
    zo = _oracle(cfg, seg, ts, X, Ps)
    assert rel_err(z, zo) <= 2e-2
    # the candidate rows are the scored outputs
    cand = sess.candidates().float().cpu().numpy()
    assert rel_err(cand, zo[sess.cand_rows]) <= 2e-2
    # a second request through the same graph (new features)
    _, X2 = _request(cfg, seg, x_stream=1)
    sess.set_request(torch.from_numpy(X2).to(dev, torch.bfloat16))
    z2 = sess.run().float().cpu().numpy()
    assert rel_err(z2, _oracle(cfg, seg, ts, X2, Ps)) <= 2e-2
    # graph replay == eager layer-by-layer forward, bit for bit
    eager = sess._forward().float().cpu().numpy()[:sess.T]
    assert np.array_equal(eager, z2)


def test_candidates_do_not_see_each_other_at_full_request_size(dev):
    """The full `infer` request (15 layers, 4096 lifelong + 100 real-time tokens, 500
    candidates): perturbing one candidate's features changes only that candidate's output
    (rule 3) and leaves the prefix rows unchanged — checked on the graph path."""
    cfg = synth.config("infer")
    seg = synth.gen_segments(cfg)
    Ps = [synth.gen_layer_params(cfg, li) for li in range(cfg["n_layers"])]
    lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
    ts, X = _request(cfg, seg)
    sess = InferenceSession(lc, [m.params_to_device(P, torch.bfloat16, dev) for P in Ps],
                            torch.bfloat16, dev, seg, ts)
    sess.set_request(torch.from_numpy(X).to(dev, torch.bfloat16))
    z1 = sess.run().clone()
    X2 = X.copy()
    j = int(sess.cand_rows[17])
    X2[j] = synth.round_bf16(X2[j] * -1.5 + 0.25)
    sess.set_request(torch.from_numpy(X2).to(dev, torch.bfloat16))
    z2 = sess.run().clone()
    diff = (z1 != z2).any(1).nonzero().flatten().cpu().numpy()
    assert diff.tolist() == [j]
