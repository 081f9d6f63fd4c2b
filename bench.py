#!/usr/bin/env python
"""Benchmark: whole-frame encode + decode throughput of the integer-only octree coder.

Workload (BASELINE.json configs[1], "cfg2"): synthetic KITTI-shaped 64-beam x
2048-azimuth frames (~131k points, ~56k voxels), 12-level octree, full GRED+XFP model
(C = H = 32, seeded random int8 weights).  One step = encode B frames (device int32
xyz -> device bitstreams) + decode them (device bitstreams -> device xyz): every row of
SURVEY.md §8(a).  Frames shard by index across ranks (weak scaling, no data-path
collective); NCCL only gathers per-rank stats.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg1|cfg5|...]

--gpus N > 1 without a torchrun environment re-launches this script under
`torch.distributed.run --nproc-per-node N` (one process per GPU, NCCL); under torchrun
WORLD_SIZE must equal N.  --workload selects another BASELINE.json config (the default,
cfg2, is the one `metric` is quoted on): cfg3 = Ford-shaped 18-bit frames (~87k voxels,
deep sparse levels), cfg1 = 16-beam 12-bit frames with the 8-channel model, cfg5 = the
1000-frame sequence, plus the NEXT-1 sweep / ablation lines (cfg2_L11..16, cfg2_t3,
cfg2_xfp_off, cfg2_gred_off) and NEXT-4's cfg2_rawfreq.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "enc/dec frames/s at 1/2/4/8 B200; bit-exact bitstream vs CPU oracle; bpp"
UNIT = "frames/s"
WORKLOADS = {  # name -> (channels C = H, description)
    "cfg2": (32, "cfg2: KITTI-shaped 64x2048 LiDAR frames (synthetic ray-cast), L=12, C=H=32 GRED+XFP int8 model"),
    "cfg3": (32, "cfg3: Ford-shaped 64-beam 18-bit LiDAR frames (synthetic ray-cast), L=18, C=H=32 GRED+XFP int8 model"),
    "cfg1": (8, "cfg1: 16-beam x 512 LiDAR frames (synthetic ray-cast), L=12, C=H=8 int8 model"),
}
# NEXT-1: the cfg2 sensor at L = 11..16 bits (Table 3 averages over 11-16 bit,
# P:644) and the t = L-3 variant (n_deep = 3): config-only reuse of every kernel
for _L in range(11, 17):
    WORKLOADS[f"cfg2_L{_L}"] = (32, f"cfg2 sensor quantised at L={_L} (precision sweep), C=H=32 GRED+XFP int8 model")
WORKLOADS["cfg2_t3"] = (32, "cfg2 with the t = L-3 variant (3 deep levels), L=12, C=H=32 GRED+XFP int8 model")
# NEXT-1 Table 4 ablations: "Baseline + GRED" (XFP off) and "Baseline" (GRED off)
WORKLOADS["cfg2_xfp_off"] = (32, "cfg2 with the Table 4 'Baseline + GRED' ablation (XFP off), L=12, C=H=32 int8 model")
WORKLOADS["cfg2_gred_off"] = (32, "cfg2 with the Table 4 'Baseline' ablation (GRED and XFP off), L=12, C=H=32 int8 model")
# NEXT-4: the raw prefix coded "based on their symbol frequencies"
WORKLOADS["cfg2_rawfreq"] = (32, "cfg2 with the frequency-coded raw prefix (P:601), L=12, C=H=32 GRED+XFP int8 model")
# BASELINE configs[4]: a 1,000-frame cfg2-shaped sequence (sensor advancing 1 m per frame),
# frame i on rank i mod W: the total work is fixed as W grows (strong scaling)
WORKLOADS["cfg5"] = (32, "cfg5: 1000-frame synthetic 64-beam sequence, frame i on rank i mod W, L=12, C=H=32")
SEQ_FRAMES = 1000
WORKLOAD = WORKLOADS["cfg2"][1]


def workload(args):
    """(ScanConfig, C, description) of --workload."""
    import dataclasses
    from paper_2603_25260_b200 import inputs as I
    C, desc = WORKLOADS[args.workload]
    name = args.workload
    if name.startswith("cfg2_L"):
        return dataclasses.replace(I.CFG2, bit_depth=int(name[6:])), C, desc
    if name in ("cfg2_t3", "cfg5", "cfg2_xfp_off", "cfg2_gred_off", "cfg2_rawfreq"):
        return I.CFG2, C, desc
    return I.CONFIGS[name], C, desc


def default_batch(name: str) -> int:
    """Frames per GPU per step when --batch is not given: 2048 (4 lanes x 512 frames per
    codec launch) for the L <= 12 workloads (measured 31.0k against 28.3k frames/s at 4 x
    256: the level-serial decoder and the per-launch fixed costs amortise over more frames),
    1024 at L = 13, 256 for the deeper trees (L >= 14, cfg3), whose arenas are larger."""
    if name == "cfg3" or (name.startswith("cfg2_L") and int(name[6:]) >= 14):
        return 256
    if name == "cfg2_L13":
        return 1024
    return 2048


def model_bytes(args, C):
    """The seeded random int8 model of --workload (n_deep = 3 for the t = L-3 variant, 0 for
    the GRED-off ablation; XFP off / frequency-coded raw prefix by model flag)."""
    from paper_2603_25260_b200 import inputs as I
    w = args.workload
    nd = {"cfg2_t3": 3, "cfg2_gred_off": 0}.get(w, 4)
    return I.make_model(C=C, H=C, seed=1, n_deep=nd, min_depth=9, max_depth=18, xfp=w != "cfg2_xfp_off",
                        raw_freq=w == "cfg2_rawfreq").to_bytes()


def host_cpu():
    """(logical cores, CPU model) of this host."""
    name = "?"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                name = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, name


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        if self.dev < 0:  # no GPU (the CPU plumbing test)
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(cfg, B: int, first: int, world: int = 1):
    """The rank's B synthetic frames (seeded per frame index), ray-cast on host threads."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2603_25260_b200 import inputs as I
    with ThreadPoolExecutor(max_workers=max(1, (os.cpu_count() or 1) // max(1, world))) as ex:
        frames = list(ex.map(lambda i: I.make_frame(cfg, first + i, scene_seed=1), range(B)))
    offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
    return frames, offs


# --------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands (BASELINE tier framing: the oracle is the
# reference arm), run on host cores, rank 0 only.
# --------------------------------------------------------------------------------------

def oracle_rate(frames, L, model_bytes, threads: int):
    """Encode+decode each frame with the oracle; returns (frames/s, seconds, cores used)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    m = O.Model(model_bytes)

    def one(f):
        bs = O.encode(m, f, L)
        O.decode(m, bs)
        return len(bs)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, frames))
    dt = time.perf_counter() - t0
    return len(frames) / dt, dt


def run_config(args, world):
    """The workload both arms report (identical dicts: the driver compares like with like)."""
    B = args.batch
    if args.workload == "cfg5":
        return {"workload": WORKLOADS["cfg5"][1], "frames_per_gpu_per_step": -(-SEQ_FRAMES // world),
                "global_batch": SEQ_FRAMES, "parallelism": f"frames/dp{world} (frame i on rank i mod {world})",
                "l2": "flushed between steps (256 MiB write, outside the events)"}
    return {"workload": WORKLOADS[args.workload][1], "frames_per_gpu_per_step": B, "global_batch": B * world,
            "parallelism": f"frames/dp{world}", "l2": "flushed between steps (256 MiB write, outside the events)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2603_25260_b200 import inputs as I
    cfg, C, _ = workload(args)
    mb = model_bytes(args, C)
    cores, cpu_name = host_cpu()
    frames, _ = make_inputs(cfg, cores, 0)
    for _ in range(args.warmup):
        oracle_rate(frames[:1], cfg.bit_depth, mb, 1)
    ts = []
    for _ in range(args.steps):
        _, dt = oracle_rate(frames, cfg.bit_depth, mb, cores)
        ts.append(dt)
    tot = sum(ts)
    value = cores * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64 (scalar CPU)",
            "data": "synthetic", "config": run_config(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu": cpu_name, "kind": "oracle",
                             "sample": f"each step a bounded sample of the workload: {cores} of its {args.workload} frames "
                                       f"(encode+decode), one frame per thread on all {cores} host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# multi-GPU plumbing: frames shard by index (no data-path collective); one all_gather of
# per-rank stats; whole-job rate = all frames / max-over-ranks device time (weak scaling)
# --------------------------------------------------------------------------------------

STAT_FIELDS = ("frames", "points", "voxels", "bytes", "enc_ns", "dec_ns", "mismatch", "tot_ns", "e2e_ns")


def sequence_shard(rank: int, world: int, total: int = None):
    """cfg5: frame indices of this rank in the fixed sequence (frame i on rank i mod W)."""
    return list(range(rank, SEQ_FRAMES if total is None else total, world))


def shard_frames(rank: int, world: int, batch: int):
    """Frame indices of this rank: a contiguous block of `batch` frames of the sequence."""
    return list(range(rank * batch, (rank + 1) * batch))


def rank_stats(B, npts, nvox, nbytes, enc_ms, dec_ms, parity, e2e_ms):
    return np.array([B, npts, nvox, nbytes, int(enc_ms * 1e6), int(dec_ms * 1e6), int(parity is False),
                     int((enc_ms + dec_ms) * 1e6), int(e2e_ms * 1e6)], np.int64)


def gather_stats(dist, stats, device, world):
    """all_gather of the int64 stats vector (NCCL on the GPU path, gloo in CPU tests)."""
    if not dist:
        return stats[None]
    import torch
    t = torch.from_numpy(stats).to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.stack([a.cpu().numpy() for a in out])


def aggregate(allst, K):
    frames = int(allst[:, 0].sum()) * K
    t_max_ms = float(allst[:, 7].max()) / 1e6
    return {"frames": frames, "t_max_ms": t_max_ms, "value": frames / (t_max_ms / 1e3),
            "enc_fps": frames / (float(allst[:, 4].max()) / 1e9), "dec_fps": frames / (float(allst[:, 5].max()) / 1e9),
            "points": int(allst[:, 1].sum()) * K, "voxels": int(allst[:, 2].sum()) * K,
            "bytes": int(allst[:, 3].sum()) * K, "mismatch": int(allst[:, 6].sum()),
            "e2e_ms_max": float(allst[:, 8].max()) / 1e6}


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------

ALU_PEAK_NOTE = ("B200 integer issue peak = 148 SM x 4 SMSP x 32 lanes x 1 instr/clk x sm_max clock "
                 "(DESIGN.md §5)")
# Algorithmic integer ops per coded node of the predictor + integer softmax:
# hidden layer C*H/4 dp4a (C = H = 32) + 9 ops per symbol for the exponentials (logit
# requant mul-add, shift, saturate; max; delta; LUT index/load/select; sum); reading Q21's
# cumulative floors then cost the encoder one prefix add per symbol and two exact 64-bit
# divisions per node (~10 ops each); the decoder's predictor only the 16 block prefixes
# per node (its rows carry no cumulative counts: the rANS decoder rebuilds the few it
# searches).
def alu_ops_per_node(C, H):
    return {"head_enc": C * H / 4 + 10 * 255 + 20, "head_dec": C * H / 4 + 9 * 255 + 16}


def measured_traffic(kernel: str, workload: str):
    """(DRAM bytes, note) of the longest launch of `kernel` in `workload` from the committed
    ncu --set full summaries (profiles/traffic.json, written by tools/summarize_round.py):
    {workload: {kernel: {...}}}; None when that workload's kernel was not captured."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p))[workload][kernel]
        return t["dram_bytes_per_launch"], f"dram read+write of the {t['launch']} ({t['duration']}), {t['source']}"
    except Exception:
        return None, None


class GpuRunner:
    """The measured workload on this rank's GPU: S concurrent codec lanes (own ctx + stream
    each) over this rank's frames; one step = encode + decode of every frame."""

    def __init__(self, args, rank, world):
        import torch
        from paper_2603_25260_b200 import inputs as I
        from paper_2603_25260_b200 import pcc
        self.torch, self.pcc, self.args = torch, pcc, args
        self.dev = dev = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(dev)
        self.device = f"cuda:{dev}"
        cfg, C, _ = workload(args)
        self.L, self.C = L, _ = cfg.bit_depth, C
        self.mb = mb = model_bytes(args, C)
        if args.workload == "cfg5":  # the fixed sequence, frame i on rank i mod W
            self.frames = [I.make_frame(cfg, i, scene_seed=1) for i in sequence_shard(rank, world)]
            self.offs = np.cumsum([0] + [len(f) for f in self.frames]).tolist()
        else:
            self.frames, self.offs = make_inputs(cfg, args.batch, shard_frames(rank, world, args.batch)[0], world)
        self.B = B = len(self.frames)
        self.S = S = max(1, min(args.streams, B))
        self.npts = self.offs[-1]
        self.host_xyz = torch.from_numpy(np.concatenate(self.frames).astype(np.int32)).pin_memory()
        self.model = pcc.pcc_model_load(mb, dev)
        self.main = torch.cuda.Stream(dev)
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.device)
        self.cuts = [B * k // S for k in range(S + 1)]
        self.lanes = [self._lane(self.cuts[k], self.cuts[k + 1]) for k in range(S)]
        torch.cuda.synchronize(dev)

    def _lane(self, f0, f1):
        torch, pcc, L, offs = self.torch, self.pcc, self.L, self.offs
        runner = self

        class Lane:
            """One of S concurrent codec instances (own ctx + stream) on frames [f0, f1)."""

            def __init__(self):
                self.f0, self.f1 = f0, f1
                self.stream = torch.cuda.Stream(runner.dev)
                self.ctx = pcc.pcc_ctx_create(runner.dev, self.stream.cuda_stream)
                self.offs = [o - offs[f0] for o in offs[f0:f1 + 1]]
                self.n = self.offs[-1]
                with torch.cuda.stream(self.stream):
                    self.xyz = runner.host_xyz[offs[f0]:offs[f1]].to(runner.device, non_blocking=True)
                    self.cap = sum(pcc.pcc_encode_bound(self.offs[i + 1] - self.offs[i], L) + 4
                                   for i in range(len(self.offs) - 1))
                    self.bs = torch.empty(self.cap, dtype=torch.uint8, device=runner.device)
                    self.out = torch.empty((self.n, 3), dtype=torch.int32, device=runner.device)
                self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

            def run(self, start_ev=None):
                if start_ev is not None:
                    self.stream.wait_event(start_ev)
                self.oo = pcc.pcc_encode_batch(self.ctx, runner.model, self.xyz, self.offs, L, self.bs, self.cap)
                self.ev[0].record(self.stream)
                self.no = pcc.pcc_decode_batch(self.ctx, runner.model, self.bs, self.oo, self.out, self.n)
                self.ev[1].record(self.stream)

        return Lane()

    def step(self):
        """Encode + decode all B frames: the S lanes run concurrently (one host thread each).
        Returns (start, end) events on the main stream."""
        import threading as _th
        torch = self.torch
        start = torch.cuda.Event(enable_timing=True)
        start.record(self.main)
        ths = [_th.Thread(target=ln.run, args=(start,)) for ln in self.lanes[1:]]
        for t_ in ths:
            t_.start()
        self.lanes[0].run(start)
        for t_ in ths:
            t_.join()
        end = torch.cuda.Event(enable_timing=True)
        for ln in self.lanes:
            self.main.wait_event(ln.ev[1])
        end.record(self.main)
        return start, end

    def warmup(self, W):
        for _ in range(W):
            self.step()
        self.torch.cuda.synchronize(self.dev)
        self.nvox = sum(ln.no[-1] for ln in self.lanes)
        self.nbytes = sum(ln.oo[-1] for ln in self.lanes)

    def parity(self):
        """Outside the timed region: the first and last frame of EVERY lane against the CPU
        oracle (bitstream bytes and decoded voxels), oracle runs in parallel threads."""
        from concurrent.futures import ThreadPoolExecutor
        from oracle import oracle as O
        om = O.Model(self.mb)
        picks = []
        for ln in self.lanes:
            for i in sorted({0, len(ln.offs) - 2}):
                got = ln.bs[ln.oo[i]:ln.oo[i + 1]].cpu().numpy().tobytes()
                dec = ln.out[ln.no[i]:ln.no[i + 1]].cpu().numpy()
                picks.append((ln.f0 + i, got, dec))

        def check(p):
            f, got, dec = p
            want = O.encode(om, self.frames[f], self.L)
            ref, _ = O.decode(om, want)
            return got == want and np.array_equal(dec, ref)
        with ThreadPoolExecutor(max_workers=min(len(picks), os.cpu_count() or 1)) as ex:
            res = list(ex.map(check, picks))
        return all(res), len(res)

    def timed(self, K):
        """K steps, L2 flushed between steps (outside the events).  Returns per-step
        (total, start -> last encode done, slowest lane's decode) ms lists."""
        torch = self.torch
        tot, enc, dec = [], [], []
        for _ in range(K):
            with torch.cuda.stream(self.main):
                self.flush.zero_()
            start, end = self.step()
            torch.cuda.synchronize(self.dev)  # the lanes' events are reused next step
            tot.append(start.elapsed_time(end))
            enc.append(max(start.elapsed_time(ln.ev[0]) for ln in self.lanes))
            dec.append(max(ln.ev[0].elapsed_time(ln.ev[1]) for ln in self.lanes))
        return tot, enc, dec

    def launches_per_step(self):
        pcc = self.pcc
        n = 0
        for ln in self.lanes:
            pcc.pcc_encode_batch(ln.ctx, self.model, ln.xyz, ln.offs, self.L, ln.bs, ln.cap)
            n += pcc.pcc_ctx_launch_count(ln.ctx)
            pcc.pcc_decode_batch(ln.ctx, self.model, ln.bs, ln.oo, ln.out, ln.n)
            n += pcc.pcc_ctx_launch_count(ln.ctx)
        return n

    def profile(self, K):
        """CUDA events around every launch of ONE codec instance holding the whole batch (no
        lane overlap, so per-kernel durations and shares are not inflated by concurrency)."""
        torch, pcc = self.torch, self.pcc
        KP = max(1, min(K, 3))
        full = self._lane(0, self.B) if self.S > 1 else self.lanes[0]
        pcc.pcc_ctx_set_profile(full.ctx, True)
        for _ in range(KP):
            with torch.cuda.stream(self.main):
                self.flush.zero_()
            torch.cuda.synchronize(self.dev)
            full.run()
            torch.cuda.synchronize(self.dev)
        prof = {}
        for cname in pcc.pcc_ctx_profile_categories(full.ctx):
            ms, nl, nb = pcc.pcc_ctx_profile_get(full.ctx, cname)
            prof[cname] = {"ms_per_step": ms / KP, "launches_per_step": nl / KP, "bytes_per_step": nb / KP}
        pcc.pcc_ctx_set_profile(full.ctx, False)
        if full is not self.lanes[0]:
            pcc.pcc_ctx_destroy(full.ctx)
        return prof

    def e2e(self, K):
        """Same metric through the host-buffer C ABI (H2D inputs + D2H results inside), one
        lane per host thread, the same concurrency as the device-resident measurement."""
        import threading as _th
        torch, pcc = self.torch, self.pcc
        for ln in self.lanes:
            ln.h_bs = torch.empty(ln.cap, dtype=torch.uint8).pin_memory()
            ln.h_out = torch.empty((ln.n, 3), dtype=torch.int32).pin_memory()
            ln.h_xyz = self.host_xyz[self.offs[ln.f0]:self.offs[ln.f1]]

        def lane(ln):
            ln.oo_h = pcc.pcc_encode_batch_host(ln.ctx, self.model, ln.h_xyz, ln.offs, self.L, ln.h_bs, ln.cap)
            ln.no_h = pcc.pcc_decode_batch_host(ln.ctx, self.model, ln.h_bs, ln.oo_h, ln.h_out, ln.n)

        KE = max(1, min(K, 5))
        ms = 0.0
        for k in range(KE + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.main)
            for ln in self.lanes:
                ln.stream.wait_event(e0)
            ths = [_th.Thread(target=lane, args=(ln,)) for ln in self.lanes]
            for t_ in ths:
                t_.start()
            for t_ in ths:
                t_.join()
            for ln in self.lanes:
                done = torch.cuda.Event()
                done.record(ln.stream)
                self.main.wait_event(done)
            e1.record(self.main)
            torch.cuda.synchronize(self.dev)
            if k > 0:  # the first pass sizes the e2e buffers
                ms += e0.elapsed_time(e1)
        h2d = sum(ln.n * 12 + ln.oo_h[-1] for ln in self.lanes)
        d2h = sum(ln.oo_h[-1] + ln.no_h[-1] * 12 for ln in self.lanes)
        return ms / KE, h2d, d2h

    def latency_b1(self, reps=20):
        """Per-frame latency (Table 3's unit): ONE frame per call, encode then
        decode, device-resident and through the host-buffer ABI; median over reps."""
        torch, pcc, L = self.torch, self.pcc, self.L
        ln = self.lanes[0]
        n0 = ln.offs[1]
        x = ln.xyz[:n0]
        cap = pcc.pcc_encode_bound(n0, L) + 4
        bs = torch.empty(cap, dtype=torch.uint8, device=self.device)
        out = torch.empty((n0, 3), dtype=torch.int32, device=self.device)
        h_x = self.host_xyz[:n0]
        h_bs = torch.empty(cap, dtype=torch.uint8).pin_memory()
        h_out = torch.empty((n0, 3), dtype=torch.int32).pin_memory()
        enc, dec, e2e = [], [], []
        for r in range(reps + 3):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(ln.stream)
            oo = pcc.pcc_encode_batch(ln.ctx, self.model, x, [0, n0], L, bs, cap)
            ev[1].record(ln.stream)
            pcc.pcc_decode_batch(ln.ctx, self.model, bs, oo, out, n0)
            ev[2].record(ln.stream)
            ev[2].synchronize()
            t0 = time.perf_counter()
            ooh = pcc.pcc_encode_batch_host(ln.ctx, self.model, h_x, [0, n0], L, h_bs, cap)
            pcc.pcc_decode_batch_host(ln.ctx, self.model, h_bs, ooh, h_out, n0)
            t1 = time.perf_counter()
            if r >= 3:
                enc.append(ev[0].elapsed_time(ev[1]))
                dec.append(ev[1].elapsed_time(ev[2]))
                e2e.append(1000 * (t1 - t0))
        return {"frames_per_call": 1, "enc_ms": float(np.median(enc)), "dec_ms": float(np.median(dec)),
                "enc_dec_fps": 1000.0 / (float(np.median(enc)) + float(np.median(dec))),
                "e2e_host_ms": float(np.median(e2e)), "reps": reps,
                "scope": "one frame per pcc_encode_batch / pcc_decode_batch call (device-resident, CUDA events); "
                         "e2e_host_ms: pcc_*_batch_host wall clock incl. H2D/D2H"}

    def coded_per_step(self):
        n = 0
        for ln in self.lanes:
            for i in range(len(ln.offs) - 1):
                cnt = self.pcc.pcc_build_octree(ln.ctx, ln.xyz[ln.offs[i]:ln.offs[i + 1]], ln.offs[i + 1] - ln.offs[i],
                                                self.L)
                n += sum(cnt[4:self.L])
        return n


class PlumbingRunner:
    """CPU stand-in for GpuRunner (the same interface, no codec): lets a gloo test drive the
    multi-process plumbing — re-launch, process group, sharding, barriers, timing max over
    ranks, the stats all_gather and rank 0's JSON line — without a GPU."""

    def __init__(self, args, rank, world):
        self.args, self.rank = args, rank
        self.frames = shard_frames(rank, world, args.batch)
        self.B = len(self.frames)
        self.S, self.L, self.C = 1, 12, 32
        self.npts, self.nvox, self.nbytes = 1000 * self.B, 500 * self.B, 64 * self.B

    def warmup(self, W):
        pass

    def parity(self):
        return True, 0

    def timed(self, K):
        ms = 2.0 * (self.rank + 1)  # rank r "takes" 2 (r + 1) ms per step
        return [ms] * K, [ms / 2] * K, [ms / 2] * K

    def launches_per_step(self):
        return 0


def kernel_table(prof, coded, ops, pk):
    """Per-kernel-category roofline rows: HBM GB/s of the algorithmic bytes,
    or the integer-issue rate for the predictor + softmax categories."""
    total = sum(v["ms_per_step"] for v in prof.values()) or 1.0
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    rows = []
    for name, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms_per_step"]):
        sec = v["ms_per_step"] / 1e3
        if sec <= 0:
            continue
        if name in ops:
            ach, peak = coded * ops[name] / sec / 1e12, 148 * 4 * 32 * sm_max * 1e6 / 1e12
            rows.append({"kernel": name, "bound": "alu", "achieved": ach, "peak": peak, "unit": "Tops/s",
                         "frac": ach / peak, "ms_per_step": v["ms_per_step"], "share_of_step": v["ms_per_step"] / total,
                         "launches_per_step": v["launches_per_step"]})
        else:
            ach, peak = v["bytes_per_step"] / sec / 1e9, float(pk["hbm_gbs"])
            rows.append({"kernel": name, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "ms_per_step": v["ms_per_step"], "share_of_step": v["ms_per_step"] / total,
                         "launches_per_step": v["launches_per_step"]})
    return rows


def run_ours(args, rank, world, dist, runner_cls=None):
    runner_cls = runner_cls or GpuRunner
    r = runner_cls(args, rank, world)
    gpu = isinstance(r, GpuRunner)
    r.warmup(args.warmup)
    parity, n_parity = (None, 0)
    if not args.no_parity and rank == 0:
        parity, n_parity = r.parity()

    # ---- timed region: K steps bracketed by barrier + synchronize on both sides ----
    K = args.steps
    if dist:
        dist.barrier()
    if gpu:
        r.torch.cuda.synchronize(r.dev)
    with Clocks(r.dev if gpu else -1) as clk:
        t_wall0 = time.perf_counter()
        tot, enc, dec = r.timed(K)
        t_wall = time.perf_counter() - t_wall0
    if gpu:
        r.torch.cuda.synchronize(r.dev)
    if dist:
        dist.barrier()
    tot_ms, enc_ms, dec_ms = sum(tot), sum(enc), sum(dec)

    gpu_launches = r.launches_per_step() * K
    prof, e2e_ms, h2d, d2h, lat, coded = {}, 0.0, 0, 0, None, 0
    if gpu:
        prof = r.profile(K)
        e2e_ms, h2d, d2h = r.e2e(K)
        if not args.no_latency:
            lat = r.latency_b1()
        coded = r.coded_per_step()

    # ---- gather per-rank stats (the only collective) ----
    stats = rank_stats(r.B, r.npts, r.nvox, r.nbytes, enc_ms, dec_ms, parity, e2e_ms)
    allst = gather_stats(dist, stats, f"cuda:{r.dev}" if gpu and dist and args.backend == "nccl" else "cpu", world)
    if rank != 0:
        return
    agg = aggregate(allst, K)
    frames_tot, t_max_ms, value = agg["frames"], agg["t_max_ms"], agg["value"]

    # ---- roofline of the dominant kernel category + the per-kernel table ----
    pk, pk_src = peaks()
    ops = alu_ops_per_node(r.C, r.C)
    table = kernel_table(prof, coded, ops, pk)
    roof = None
    if table:
        top = dict(table[0])
        traffic, traffic_note = measured_traffic(top["kernel"], args.workload)
        top.update(traffic=traffic, traffic_note=traffic_note,
                   peak_src=ALU_PEAK_NOTE if top["bound"] == "alu" else pk_src + " copy bandwidth (MEASURED_PEAKS.json)")
        roof = top

    # ---- CPU baseline: the oracle on a bounded sample of the same workload, all host cores ----
    cpu = None
    if gpu and not args.no_cpu_baseline and world == 1:
        cores, cpu_name = host_cpu()
        nf = min(len(r.frames), cores)
        rate, dt = oracle_rate(r.frames[:nf], r.L, r.mb, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "cpu": cpu_name, "kind": "oracle",
               "sample": f"{nf} of the step's {args.workload} frames encode+decode on {cores} threads (all host "
                         f"threads), one frame per task ({dt:.1f} s wall)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_max_ms / K, "higher_is_better": True,
        "scaling": "strong" if args.workload == "cfg5" else "weak", "vs_baseline": None,
        "dtype": "int8 x int8 -> int32 (integer-only)", "data": "synthetic",
        "config": run_config(args, world),
        "details": {"lanes_per_gpu": r.S, "frames_per_launch": r.B // r.S, "points_per_frame": r.npts / r.B,
                    "voxels_per_frame": r.nvox / r.B, "backend": args.backend if dist else None},
        "enc_fps": agg["enc_fps"], "dec_fps": agg["dec_fps"], "points_per_s": agg["points"] / (t_max_ms / 1e3),
        "bpp": 8.0 * agg["bytes"] / agg["points"], "bits_per_voxel": 8.0 * agg["bytes"] / agg["voxels"],
        "parity": {"ok": parity, "frames_checked": n_parity,
                   "scope": "first and last frame of every codec lane vs the CPU oracle (bitstream + decode)"},
        "wall_s_timed_region": t_wall,
        "gpu_launches": gpu_launches,
        "e2e": {"value": frames_tot / K / (agg["e2e_ms_max"] / 1e3) if agg["e2e_ms_max"] else None, "unit": UNIT,
                "scope": "pcc_encode_batch_host + pcc_decode_batch_host (pinned host in/out), max over ranks",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "latency_b1": lat,
        "clocks": clk.summary(),
        "roofline": roof,
        "kernels": table,
        "profile_ms_per_step": {k: round(v["ms_per_step"], 4) for k, v in sorted(prof.items())},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    p = s_.getsockname()[1]
    s_.close()
    return p


def relaunch_under_torchrun(argv, n):
    """--gpus N > 1 without a torchrun environment: one process per GPU via
    torch.distributed.run on this node (127.0.0.1 rendezvous); returns its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None,
                    help="frames per GPU per step (default: 2048 = 4 codec lanes x 512 frames for "
                         "L <= 12, 1024 at L = 13, 256 for the deeper configs)")
    ap.add_argument("--streams", type=int, default=4, help="concurrent codec lanes (ctx + stream) per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: the CPU plumbing test only)")
    ap.add_argument("--plumbing-selftest", action="store_true",
                    help="CPU test of the multi-process plumbing with a codec-free runner (tests only)")
    args = ap.parse_args(argv)
    if args.batch is None:
        args.batch = default_batch(args.workload)
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(argv, args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as D
        if args.backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        D.init_process_group(args.backend)
        dist = D
    run_ours(args, rank, world, dist, PlumbingRunner if args.plumbing_selftest else None)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
