"""NEXT-3 HRCS report (Fig.1c) on the synthetic configs, through the C ABI.

usage (GPU box): python tools/hrcs_report.py [--frames 64] > gpurun_out/hrcs.txt
Prints, per config, the mean node count and mean occupied 26-neighbours per depth over
the frames, and the device time of one pcc_hrcs_stats call (CUDA events, after warm-up).
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_25260_b200 import inputs as I  # noqa: E402
from paper_2603_25260_b200 import pcc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    a = ap.parse_args()
    ctx = pcc.pcc_ctx_create(0, torch.cuda.current_stream().cuda_stream)
    for name in ("cfg1", "cfg2", "cfg3"):
        sc = I.CONFIGS[name]
        frames = I.make_frames(sc, a.frames, first=0)
        offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
        x = torch.from_numpy(np.concatenate(frames).astype(np.int32)).cuda()
        L = sc.bit_depth
        for _ in range(3):
            nodes, nsum = pcc.pcc_hrcs_stats(ctx, x, offs, L)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            nodes, nsum = pcc.pcc_hrcs_stats(ctx, x, offs, L)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        mean_nodes = nodes.astype(np.float64).mean(0)
        mean_nbr = (nsum.astype(np.float64) / np.maximum(nodes, 1)).mean(0)
        print(f"== {name} ({sc.name}), {a.frames} frames, L = {L}: {ms:.3f} ms per call "
              f"({a.frames / ms * 1e3:.0f} frames/s, host sync included)")
        print("depth  mean_nodes  mean_occupied_26_neighbours")
        for d in range(L + 1):
            print(f"{d:5d}  {mean_nodes[d]:10.1f}  {mean_nbr[d]:8.3f}")
    pcc.pcc_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
