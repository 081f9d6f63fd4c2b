"""One warm-up step + N measured steps of the bench workload (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_25260_b200 import inputs as I
from paper_2603_25260_b200 import pcc

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--cfg", default="cfg2")
a = ap.parse_args()
cfg = I.CONFIGS[a.cfg]
C = cfg.channels
mb = I.make_model(C=C, H=C, seed=1, min_depth=9, max_depth=18).to_bytes()
frames = I.make_frames(cfg, a.batch, 0)
offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
codec = pcc.Codec(mb, 0)
x = torch.from_numpy(np.concatenate(frames)).cuda()
for k in range(1 + a.steps):
    bs, oo = codec.encode_frames(x, offs, cfg.bit_depth)
    out, no = codec.decode_frames(bs, oo, offs[-1])
torch.cuda.synchronize()
enc_l = None
print("ok", oo[-1], no[-1])
