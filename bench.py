#!/usr/bin/env python
"""Benchmark: whole-frame encode + decode throughput of the integer-only octree coder.

Workload (BASELINE.json configs[1], "cfg2"): synthetic KITTI-shaped 64-beam x
2048-azimuth frames (~131k points, ~56k voxels), 12-level octree, full GRED+XFP model
(C = H = 32, seeded random int8 weights).  One step = encode B frames (device int32
xyz -> device bitstreams) + decode them (device bitstreams -> device xyz): every row of
SURVEY.md §8(a).  Frames shard by index across ranks (weak scaling, no data-path
collective); NCCL only gathers per-rank stats.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg1]

--workload selects another BASELINE.json config (the default, cfg2, is the one `metric`
is quoted on): cfg3 = Ford-shaped 18-bit frames (~87k voxels, deep sparse levels), cfg1 =
16-beam 12-bit frames with the 8-channel model.
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
    if name in ("cfg2_t3", "cfg5"):
        return I.CFG2, C, desc
    return I.CONFIGS[name], C, desc


def default_batch(name: str) -> int:
    """Frames per GPU per step when --batch is not given: 1024 (4 lanes x 256 frames) where
    a lane's arena fits comfortably (L <= 13), 256 for the deeper trees (L >= 14, cfg3)."""
    deep = name == "cfg3" or (name.startswith("cfg2_L") and int(name[6:]) >= 14)
    return 256 if deep else 1024


def model_bytes(args, C):
    """The seeded random int8 model of --workload (n_deep = 3 for the t = L-3 variant)."""
    from paper_2603_25260_b200 import inputs as I
    nd = 3 if args.workload == "cfg2_t3" else 4
    return I.make_model(C=C, H=C, seed=1, n_deep=nd, min_depth=9, max_depth=18).to_bytes()


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


def make_inputs(cfg, B: int, first: int):
    from paper_2603_25260_b200 import inputs as I
    frames = I.make_frames(cfg, B, first=first, scene_seed=1)
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
    cores = max(1, min(os.cpu_count() or 1, 8))
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
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"each step a bounded sample of the workload: {cores} of its {args.workload} frames "
                                       f"(encode+decode), one frame per thread"},
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
# divisions per node (~10 ops each); the decoder's predictor only stores each symbol's LUT
# index (10 per symbol) and the 16 block prefixes: its rows carry no cumulative counts
# (the rANS decoder rebuilds the few it searches).
def alu_ops_per_node(C, H):
    return {"head_enc": C * H / 4 + 10 * 255 + 20, "head_dec": C * H / 4 + 10 * 255 + 16}


def measured_traffic(kernel: str):
    """(DRAM bytes, note) of the longest launch of `kernel` from the committed ncu --set full
    summary (profiles/traffic.json, written by tools/summarize_round.py), if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p))[kernel]
        return t["dram_bytes_per_launch"], f"dram read+write of the {t['launch']} ({t['duration']}), {t['source']}"
    except Exception:
        return None, None


def run_ours(args, rank, world, dist):
    import torch
    from paper_2603_25260_b200 import inputs as I
    from paper_2603_25260_b200 import pcc

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    cfg, C, _ = workload(args)
    L = cfg.bit_depth
    mb = model_bytes(args, C)
    if args.workload == "cfg5":  # the fixed sequence, frame i on rank i mod W
        frames = [I.make_frame(cfg, i, scene_seed=1) for i in sequence_shard(rank, world)]
        offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
        B = len(frames)
    else:
        B = args.batch
        frames, offs = make_inputs(cfg, B, shard_frames(rank, world, B)[0])
    S = max(1, min(args.streams, B))
    npts = offs[-1]
    host_xyz = torch.from_numpy(np.concatenate(frames).astype(np.int32)).pin_memory()
    model = pcc.pcc_model_load(mb, dev)
    main = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    class Lane:
        """One of S concurrent codec instances (own ctx + stream) on a slice of the frames."""

        def __init__(self, f0, f1):
            self.stream = torch.cuda.Stream(dev)
            self.ctx = pcc.pcc_ctx_create(dev, self.stream.cuda_stream)
            self.offs = [o - offs[f0] for o in offs[f0:f1 + 1]]
            self.n = self.offs[-1]
            with torch.cuda.stream(self.stream):
                self.xyz = host_xyz[offs[f0]:offs[f1]].to(f"cuda:{dev}", non_blocking=True)
                self.cap = sum(pcc.pcc_encode_bound(self.offs[i + 1] - self.offs[i], L) + 4
                               for i in range(len(self.offs) - 1))
                self.bs = torch.empty(self.cap, dtype=torch.uint8, device=f"cuda:{dev}")
                self.out = torch.empty((self.n, 3), dtype=torch.int32, device=f"cuda:{dev}")
            self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

        def run(self, start_ev=None):
            if start_ev is not None:
                self.stream.wait_event(start_ev)
            self.oo = pcc.pcc_encode_batch(self.ctx, model, self.xyz, self.offs, L, self.bs, self.cap)
            self.ev[0].record(self.stream)
            self.no = pcc.pcc_decode_batch(self.ctx, model, self.bs, self.oo, self.out, self.n)
            self.ev[1].record(self.stream)

    cuts = [B * k // S for k in range(S + 1)]
    lanes = [Lane(cuts[k], cuts[k + 1]) for k in range(S)]
    torch.cuda.synchronize(dev)
    import threading as _th

    def step(timed=False):
        """Encode + decode all B frames: the S lanes run concurrently (one host thread each)."""
        start = torch.cuda.Event(enable_timing=True)
        start.record(main)
        ths = [_th.Thread(target=ln.run, args=(start,)) for ln in lanes[1:]]
        for t_ in ths:
            t_.start()
        lanes[0].run(start)
        for t_ in ths:
            t_.join()
        end = torch.cuda.Event(enable_timing=True)
        for ln in lanes:
            main.wait_event(ln.ev[1])
        end.record(main)
        return start, end

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    nvox = sum(ln.no[-1] for ln in lanes)
    nbytes = sum(ln.oo[-1] for ln in lanes)

    # parity sample (outside the timed region): frame 0 vs the CPU oracle, and round trip
    parity = None
    if not args.no_parity and rank == 0:
        from oracle import oracle as O
        l0 = lanes[0]
        got = l0.bs[l0.oo[0]:l0.oo[1]].cpu().numpy().tobytes()
        want = O.encode(O.Model(mb), frames[0], L)
        dec = l0.out[l0.no[0]:l0.no[1]].cpu().numpy()
        ref, _ = O.decode(O.Model(mb), want)
        parity = bool(got == want and np.array_equal(dec, ref))

    # ---- timed region: K steps, L2 flushed between steps (outside the events) ----
    K = args.steps
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = []
    with Clocks(dev) as clk:
        t_wall0 = time.perf_counter()
        for k in range(K):
            with torch.cuda.stream(main):
                flush.zero_()
            start, end = step(True)
            evs.append((start, end, [(ln.ev[0], ln.ev[1]) for ln in lanes]))
            torch.cuda.synchronize(dev)  # lanes' events are reused next step
            evs[-1] = (start.elapsed_time(end), max(start.elapsed_time(a_) for a_, _ in evs[-1][2]),
                       max(a_.elapsed_time(b_) for a_, b_ in evs[-1][2]))
        t_wall = time.perf_counter() - t_wall0
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    tot_ms = sum(e[0] for e in evs)
    enc_ms = sum(e[1] for e in evs)  # start -> last lane's encode done
    dec_ms = sum(e[2] for e in evs)  # slowest lane's decode
    # own-kernel launches per step (counted by the library, per ctx)
    step()
    torch.cuda.synchronize(dev)
    gpu_launches = 0
    for ln in lanes:
        pcc.pcc_encode_batch(ln.ctx, model, ln.xyz, ln.offs, L, ln.bs, ln.cap)
        gpu_launches += pcc.pcc_ctx_launch_count(ln.ctx)
        pcc.pcc_decode_batch(ln.ctx, model, ln.bs, ln.oo, ln.out, ln.n)
        gpu_launches += pcc.pcc_ctx_launch_count(ln.ctx)
    gpu_launches *= K

    # ---- profiled pass: CUDA events around every launch of ONE codec instance holding the
    #      whole batch (no lane overlap, so per-kernel durations and shares are not
    #      inflated by concurrent streams) ----
    KP = max(1, min(K, 3))
    full = Lane(0, B) if S > 1 else lanes[0]
    pcc.pcc_ctx_set_profile(full.ctx, True)
    for _ in range(KP):
        with torch.cuda.stream(main):
            flush.zero_()
        torch.cuda.synchronize(dev)
        full.run()
        torch.cuda.synchronize(dev)
    prof = {}
    for cname in pcc.pcc_ctx_profile_categories(full.ctx):
        ms, nl, nb = pcc.pcc_ctx_profile_get(full.ctx, cname)
        prof[cname] = {"ms_per_step": ms / KP, "launches_per_step": nl / KP, "bytes_per_step": nb / KP}
    pcc.pcc_ctx_set_profile(full.ctx, False)
    if full is not lanes[0]:
        pcc.pcc_ctx_destroy(full.ctx)
        del full
    prof_total = sum(v["ms_per_step"] for v in prof.values())

    # ---- e2e through the host-buffer C ABI (H2D inputs + D2H results inside), one lane
    #      per host thread, same concurrency as the device-resident measurement ----
    for ln in lanes:
        ln.h_bs = torch.empty(ln.cap, dtype=torch.uint8).pin_memory()
        ln.h_out = torch.empty((ln.n, 3), dtype=torch.int32).pin_memory()
        ln.h_xyz = host_xyz[offs[cuts[lanes.index(ln)]]:offs[cuts[lanes.index(ln) + 1]]]

    def e2e_lane(ln):
        ln.oo_h = pcc.pcc_encode_batch_host(ln.ctx, model, ln.h_xyz, ln.offs, L, ln.h_bs, ln.cap)
        ln.no_h = pcc.pcc_decode_batch_host(ln.ctx, model, ln.h_bs, ln.oo_h, ln.h_out, ln.n)

    KE = max(1, min(K, 5))
    e2e_ms = 0.0
    for k in range(KE + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for ln in lanes:
            ln.stream.wait_event(e0)
        ths = [_th.Thread(target=e2e_lane, args=(ln,)) for ln in lanes]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        for ln in lanes:
            done = torch.cuda.Event()
            done.record(ln.stream)
            main.wait_event(done)
        e1.record(main)
        torch.cuda.synchronize(dev)
        if k > 0:  # the first pass sizes the e2e buffers
            e2e_ms += e0.elapsed_time(e1)
    e2e_ms /= KE
    h2d = sum(ln.n * 12 + ln.oo_h[-1] for ln in lanes)
    d2h = sum(ln.oo_h[-1] + ln.no_h[-1] * 12 for ln in lanes)
    d_xyz_list = [(ln.xyz, ln.offs) for ln in lanes]

    # coded symbols per step (levels R..L-1 of every frame), for per-node op counts
    coded_per_step = 0
    for xyz_l, offs_l in d_xyz_list:
        for i in range(len(offs_l) - 1):
            cnt = pcc.pcc_build_octree(lanes[0].ctx, xyz_l[offs_l[i]:offs_l[i + 1]], offs_l[i + 1] - offs_l[i], L)
            coded_per_step += sum(cnt[4:L])
    ops_per_node = alu_ops_per_node(C, C)

    # ---- gather per-rank stats (the only collective) ----
    stats = rank_stats(B, npts, nvox, nbytes, enc_ms, dec_ms, parity, e2e_ms)
    allst = gather_stats(dist, stats, f"cuda:{dev}", world)
    if rank != 0:
        return
    agg = aggregate(allst, K)
    frames_tot, t_max_ms, value = agg["frames"], agg["t_max_ms"], agg["value"]
    enc_fps, dec_fps, pts_tot, e2e_ms_max = agg["enc_fps"], agg["dec_fps"], agg["points"], agg["e2e_ms_max"]

    # ---- roofline of the dominant kernel category ----
    pk, pk_src = peaks()
    top = max(prof.items(), key=lambda kv: kv[1]["ms_per_step"]) if prof else (None, None)
    roof = None
    if top[0]:
        name, v = top
        sec = v["ms_per_step"] / 1e3
        traffic, traffic_note = measured_traffic(name)
        if name in ops_per_node:
            # integer-ALU bound: algorithmic ops per coded node x coded nodes per step
            sm_max = float(pk.get("sm_max_mhz", 1965.0))
            achieved = coded_per_step * ops_per_node[name] / sec / 1e12
            peak = 148 * 4 * 32 * sm_max * 1e6 / 1e12
            roof = {"kernel": name, "bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note, "peak_src": ALU_PEAK_NOTE,
                    "launches_per_step": v["launches_per_step"], "share_of_step": v["ms_per_step"] / prof_total}
        else:
            achieved = v["bytes_per_step"] / sec / 1e9
            peak = float(pk["hbm_gbs"])
            roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note,
                    "peak_src": pk_src + " copy bandwidth",
                    "launches_per_step": v["launches_per_step"], "share_of_step": v["ms_per_step"] / prof_total}

    # ---- CPU baseline: the oracle on a bounded sample of the same workload ----
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cores = max(1, min(os.cpu_count() or 1, 8))
        nf = min(len(frames), 8)
        rate, dt = oracle_rate(frames[:nf], L, mb, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{nf} of the step's {args.workload} frames encode+decode on {cores} threads, one frame "
                         f"per task ({dt:.1f} s wall)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_max_ms / K, "higher_is_better": True,
        "scaling": "strong" if args.workload == "cfg5" else "weak", "vs_baseline": None,
        "dtype": "int8 x int8 -> int32 (integer-only)", "data": "synthetic",
        "config": run_config(args, world),
        "details": {"lanes_per_gpu": S, "frames_per_launch": B // S, "points_per_frame": npts / B,
                    "voxels_per_frame": nvox / B},
        "enc_fps": enc_fps, "dec_fps": dec_fps, "points_per_s": pts_tot / (t_max_ms / 1e3),
        "bpp": 8.0 * nbytes / npts, "bits_per_voxel": 8.0 * nbytes / nvox,
        "parity_sample_frame0": parity, "wall_s_timed_region": t_wall,
        "gpu_launches": gpu_launches,
        "e2e": {"value": frames_tot / K / (e2e_ms_max / 1e3) if e2e_ms_max else None, "unit": UNIT,
                "scope": "pcc_encode_batch_host + pcc_decode_batch_host (pinned host in/out), max over ranks",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "clocks": clk.summary(),
        "roofline": roof,
        "profile_ms_per_step": {k: round(v["ms_per_step"], 4) for k, v in sorted(prof.items())},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None,
                    help="frames per GPU per step (default: 1024 = 4 codec lanes x 256 frames for "
                         "L <= 13, 256 for the deeper configs, whose per-lane arenas are larger)")
    ap.add_argument("--streams", type=int, default=4, help="concurrent codec lanes (ctx + stream) per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    if args.batch is None:
        args.batch = default_batch(args.workload)
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as D
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        D.init_process_group("nccl")
        dist = D
    run_ours(args, rank, world, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
