"""Phase timing of the tcgen05 predictor kernel (dev only): builds libpcc with -DPCC_TRACE."""
import ctypes as ct
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
so = os.path.join(ROOT, "tools", "micro", "libpcc_trace.so")
src = sorted(glob.glob(os.path.join(ROOT, "paper_2603_25260_b200", "csrc", "*.cu")))
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "-DPCC_TRACE", "-o", so, *src, "-lcuda"])
os.environ["PCC_LIB"] = so
sys.path.insert(0, ROOT)
import numpy as np  # noqa
import torch  # noqa
from paper_2603_25260_b200 import inputs as I, pcc  # noqa

lib = ct.CDLL(so)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = I.CFG2
mb = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18).to_bytes()
frames = I.make_frames(cfg, B, 0)
offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
codec = pcc.Codec(mb, 0)
x = torch.from_numpy(np.concatenate(frames)).cuda()
bs, oo = codec.encode_frames(x, offs, 12)
codec.decode_frames(bs, oo, offs[-1])
torch.cuda.synchronize()
buf = (ct.c_ulonglong * 16)()
lib.pcc_trace_head(buf, 1)
bs, oo = codec.encode_frames(x, offs, 12)
codec.decode_frames(bs, oo, offs[-1])
torch.cuda.synchronize()
lib.pcc_trace_head(buf, 0)
names = ["hidden+bias+bar", "mma wait", "pass1+bar", "pass2+bars", "pass3 (+stage)", "tail/write-out", "end barrier"]
for mode in (0, 1):
    v = buf[8 * mode: 8 * mode + 7]
    tot = sum(v) or 1
    print("encoder" if mode == 0 else "decoder")
    for i, nme in enumerate(names):
        print(f"  {nme:18s} {v[i] / 1e6:10.2f} Mcyc  {100 * v[i] / tot:5.1f}%")
