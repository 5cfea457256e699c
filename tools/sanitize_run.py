#!/usr/bin/env python
"""Small workload for compute-sanitizer (tools/gpu_sanitize.sh): one bf16 layer forward +
backward on the `parity` batch through every tensor-core backward path (MTGR_ATTN_BWD = kv,
stored, fused_dk; MTGR_ATTN_RECOMPUTE=1), the fp32 `toy` layer, and the attention-only calls."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2505_18654_b200 as m
    from tests.fixtures import make_batch
    dev = torch.device("cuda:0")
    path = os.environ.get("MTGR_ATTN_BWD", "kv") + ("+recompute" if os.environ.get("MTGR_ATTN_RECOMPUTE") == "1" else "")
    for name in sys.argv[1:] or ["toy", "parity"]:
        cfg, seg, ts, X, dZ, P = make_batch(name)
        dt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
        jb = m.JaggedBatch.build(seg, ts, dev)
        lc = m.layer_cfg(cfg["d"], cfg["H"], cfg["groups"])
        st = m.HstuStack(lc, [m.params_to_device(P, dt, dev)], dt, dev)
        st.bind(jb)
        z = st.forward(torch.from_numpy(X).to(dev, dt))
        dx = st.backward(torch.from_numpy(dZ).to(dev, dt))
        torch.cuda.synchronize()
        print(f"sanitize_run {name} path={path}: z {float(z.float().abs().sum()):.4e} dx {float(dx.float().abs().sum()):.4e}", flush=True)


if __name__ == "__main__":
    main()
