"""Development diagnostic: decoder rows of a GPU decode vs the oracle's tensors, field by field."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I, pcc
from test_gpu_parity import gpu_decode
C = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mobj = I.make_model(C=C, H=C, seed=1, min_depth=9, max_depth=18)
mb = mobj.to_bytes(); om = O.Model(mb)
pts = I.make_frame(I.CFG1)
D = O.Dump(); bs = O.encode(om, pts, 12, D)
ctx = pcc.pcc_ctx_create(0, torch.cuda.current_stream().cuda_stream)
m = pcc.pcc_model_load(mb, 0)
pcc.pcc_ctx_set_debug(ctx, True)
try:
    gpu_decode(pcc, ctx, m, [bs], len(pts)); print("decode ok")
except pcc.PCCError as e:
    print("decode error", e.name)
L = 12; Dd = L - 1 - mobj.n_deep; H = C
for d in range(4, 12):
    r = pcc.pcc_debug_tensor(ctx, f"cdf/{d}")
    if r is None: print(d, "no rows"); continue
    print(d, "cdf bytes", len(r), "oracle nodes", D.get(f"key/{d}", np.uint64).size)
    if len(r) == 0: continue
    raw = np.frombuffer(r, np.uint8).reshape(-1, 112)
    hd = mobj.shallow[d].head if d <= Dd else mobj.deep[d - Dd - 1].head
    hdr = raw[:, :72].copy().view(np.uint32).astype(np.int64)
    a = raw[:, 80:80 + H].copy().view(np.int8).astype(np.int64)
    wa = D.get(f"a/{d}", np.int8).reshape(-1, H).astype(np.int64)
    z = wa @ hd.W2.astype(np.int64).T + hd.b2.astype(np.int64)
    m_l, r_l = hd.rq_logit.m_pos, hd.rq_logit.r
    l = np.clip((z * m_l + ((1 << (r_l - 1)) if r_l else 0)) >> r_l, -(1 << 24), 1 << 24)
    mu = l.max(1); dl = mu[:, None] - l
    lut = I.exp_lut().astype(np.int64)
    e = np.where(dl < 4096, lut[np.minimum(dl, 4095) >> 2], 0)
    E = np.concatenate([np.zeros((e.shape[0], 1), np.int64), np.cumsum(e, 1)], 1)
    print(d, "rows", raw.shape[0], "a bad", int((a != wa).any(1).sum()), "S bad", int((hdr[:, 0] != E[:, 255]).sum()),
          "mu bad", int((hdr[:, 2].astype(np.uint32).view(np.int32) != mu).sum()), "E bad", int((hdr[:, 3:18] != E[:, 16:241:16]).any(1).sum()),
          "code", (lambda g: None if g is None else int((np.frombuffer(g, np.uint8) != D.get(f"code/{d}", np.uint8)).sum()))(pcc.pcc_debug_tensor(ctx, f"code/{d}")))
    if (a != wa).any():
        i = int(np.flatnonzero((a != wa).any(1))[0]); print("  row", i, "a", a[i].tolist(), "want", wa[i].tolist())
    if (hdr[:, 2].astype(np.uint32).view(np.int32) != mu).any():
        i = int(np.flatnonzero(hdr[:, 2].astype(np.uint32).view(np.int32) != mu)[0]); print("  row", i, "hdr", hdr[i, :4].tolist(), "mu", mu[i], "S", E[i,255])
