"""compute-sanitizer target: encode + decode one cfg1 frame (C = 8 and C = 32 models) and a
frame of every Table 4 variant through the C ABI, checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I
from paper_2603_25260_b200 import pcc

pts = I.make_frame(I.CFG1)
for C, kw in [(8, {}), (32, {}), (32, dict(xfp=False)), (32, dict(n_deep=0)), (8, dict(raw_freq=True))]:
    mb = I.make_model(C=C, H=C, seed=1, min_depth=9, max_depth=12, **kw).to_bytes()
    om = O.Model(mb)
    codec = pcc.Codec(mb, 0)
    out, oo = codec.encode_frames(torch.from_numpy(pts).cuda(), [0, len(pts)], 12)
    bs = out[:oo[1]].cpu().numpy().tobytes()
    assert bs == O.encode(om, pts, 12), (C, kw)
    xyz, no = codec.decode_frames(out, oo, len(pts))
    assert np.array_equal(xyz[:no[1]].cpu().numpy(), O.decode(om, bs)[0]), (C, kw)
    codec.close()
    print("ok", C, kw, len(bs), flush=True)
