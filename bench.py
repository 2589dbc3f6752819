#!/usr/bin/env python
"""Benchmark: learner frames/sec (+ InferenceServer actions/sec) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Workload (BASELINE.json): config C3 -- Pommerman-shaped obs (11x11x16 = 1936 binary
planes), MLP 1936-256-256-(6,1), PPO + GAE, T=32, a draw of B=4096 segments, Adam.  One
step = one Learner::TrainStep on every rank: returns, loss fwd/bwd, NCCL gradient
allreduce (per-layer buckets overlapped with the backward), optimizer.  N>1 is launched
by torchrun, one rank per GPU.  --scaling weak (default): B=4096 segments per learner
shard, HyperParams::batch_size being per shard in the reference (learner.cpp:108), so G
ranks consume a G x 4096-segment draw per step; at N>1 the strong-scaling figure (one
4096-segment draw split over the G ranks) is measured in the same run and
reported beside it (`strong_scaling`).  --scaling strong makes the split draw the value.

* value   : frames/s with the batch already resident in HBM (whole job, all ranks),
            timed with CUDA events on the learner's stream, max over ranks.
* e2e     : the same through the C ABI with HOST buffers (pinned): the per-step H2D
            of the shard's segments and the D2H of the step statistics are inside
            the timed region.
* roofline: the dominant kernel (layer-1 forward GEMM, tcgen05 kind::tf32) --
            algorithmic FLOPs / its own CUDA-event time, against MEASURED_PEAKS.json.
* cpu_baseline / --impl reference: the reference's own Learner::TrainStep
            (oracle/_ref, compiled from the reference sources) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region (NVML)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.stop_flag = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_flag.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_flag.set()
        if self.nv:
            self.t.join()

    def result(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def oracle_policy_cpu(c4, n=2048, reps=2):
    """The InfServer's model on the CPU: the fp64 oracle's policy forward (the reference's
    policy::Distribution / ValueEstimate arithmetic extended to the MLP family, on the
    oracle's thread pool) over `n` observations of the C4 shape.  A port: the reference's
    InfServer serves linear / tabular blobs only (types.hpp:14)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ffi import Oracle, Shape
    orc = Oracle()
    shape = Shape(2, c4.obs_dim, c4.n_actions, c4.hidden)
    p = orc.init_params(shape, 0.05, 3)
    obs = np.random.default_rng(5).standard_normal((n, c4.obs_dim))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.forward(shape, p, obs)
        ts.append(time.perf_counter() - t0)
    return {"value": n / min(ts), "unit": "actions/s", "cores": min(64, os.cpu_count() or 1),
            "kind": "port",
            "sample": f"fp64 oracle policy forward (MLP {c4.obs_dim}-"
                      f"{'-'.join(map(str, c4.hidden))}-({c4.n_actions},1)) on {n} observations, "
                      f"best of {reps}"}


# ---------------------------------------------------------------------------
def oracle_mlp_cpu(cfg, segments=64, reps=2):
    """The same model on the CPU: the fp64 oracle's learner step (oracle/tlg_oracle.cpp --
    the reference's rlmath/policy arithmetic extended to the MLP family, std::thread over
    16 fixed sample chunks) on a `segments` x T slice of the config (>= 2048 frames).
    A port, not the reference (which has no MLP family, types.hpp:14)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ffi import Hyper, Oracle, Segments, Shape
    from paper_2011_12895_b200.synth import make_segments
    orc = Oracle()
    T, D, A = cfg.unroll_len, cfg.obs_dim, cfg.n_actions
    shape = Shape(2, D, A, cfg.hidden)
    p = orc.init_params(shape, 0.05, 3)
    hp = Hyper(learning_rate=3e-4, batch_size=segments, unroll_len=T)
    algo = {"ppo": 0, "vtrace": 1, "ppo_vtrace": 2}[cfg.algo]
    b = make_segments(segments, T, D, A, seed=77, obs_kind=cfg.obs_kind)
    seg = Segments(b.obs.astype(np.float64), b.action.astype(np.uint32),
                   b.reward.astype(np.float64), b.behavior_logp.astype(np.float64),
                   b.value_est.astype(np.float64), b.done, b.bootstrap.astype(np.float64),
                   b.valid_steps.astype(np.uint32))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.learner_step(shape, p, hp, algo, [seg])
        ts.append(time.perf_counter() - t0)
    frames = int(b.valid_steps.sum())
    return {"value": frames / min(ts), "unit": "frames/s",
            "cores": min(16, os.cpu_count() or 1), "kind": "port",
            "sample": f"fp64 oracle learner step (same MLP {D}-{'-'.join(map(str, cfg.hidden))}"
                      f"-({A},1), {cfg.algo}) on {segments} segments x T={T} = {frames} "
                      f"frames, best of {reps}"}


def reference_cpu(cfg, seconds=12.0, steps=None, warmup=0, segs_per_shard=None, shards=None):
    """The reference's own Learner::TrainStep (linear_softmax: the only policy family the
    reference has, types.hpp:14) at the config's obs/A/T, num_shards = host cores, on a
    bounded sample (segs_per_shard segments per shard per step)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ffi import Hyper, RefLearner, RefLib, Segments
    from paper_2011_12895_b200.synth import make_segments
    ref = RefLib()
    cores = shards or os.cpu_count() or 1
    T, D, A = cfg.unroll_len, cfg.obs_dim, cfg.n_actions
    if segs_per_shard is None:
        # keep one step's fp64 AoS segments around ~64 MB
        segs_per_shard = max(1, min(cfg.batch_size, int(64e6 / (T * D * 8 * cores))))
    hp = Hyper(learning_rate=3e-4, batch_size=segs_per_shard, unroll_len=T, max_reuse=1)
    algo = 0 if cfg.algo == "ppo" else 1
    lrn = RefLearner(ref, ShapeLin(D, A), hp, init_scale=0.05, num_shards=cores, algo=algo,
                     publish_interval=1 << 30, replay_capacity=1 << 20, seed=7)
    draw = segs_per_shard * cores
    times, frames = [], []
    k = 0
    t_start = time.perf_counter()
    while True:
        b = make_segments(draw, T, D, A, seed=5000 + k, obs_kind=cfg.obs_kind)
        seg = Segments(b.obs.astype(np.float64), b.action.astype(np.uint32),
                       b.reward.astype(np.float64), b.behavior_logp.astype(np.float64),
                       b.value_est.astype(np.float64), b.done, b.bootstrap.astype(np.float64),
                       b.valid_steps.astype(np.uint32))
        lrn.push(seg)
        c0 = lrn.consumed()
        t0 = time.perf_counter()
        assert lrn.train_step()
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
            frames.append(lrn.consumed() - c0)
        k += 1
        if steps is not None:
            if k >= warmup + steps:
                break
        elif time.perf_counter() - t_start > seconds and len(times) >= 2:
            break
    fps = float(np.sum(frames) / np.sum(times))
    sample = (f"reference Learner::TrainStep, linear_softmax obs {D} A {A} T {T}, "
              f"{cores} shards x {segs_per_shard} segments per step, {len(times)} steps")
    return fps, cores, sample, float(np.mean(times))


def ShapeLin(D, A):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ffi import Shape
    return Shape(1, D, A)


def run_reference_arm(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    try:
        fps, cores, sample, ms = reference_cpu(cfg, steps=args.steps, warmup=args.warmup)
    except Exception as e:  # pragma: no cover - reported, not raised
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return 0
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "note": cfg.note, "policy": "linear_softmax (reference)"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


METRIC = "learner frames/sec at 1/2/4/8 B200 + InferenceServer actions/sec vs CPU ref"


def _ncu_traffic(kernel="fwd1"):
    """dram__bytes_read + dram__bytes_write of the dominant kernel per launch, from the
    committed ncu --set full capture (profiles/r02_<kernel>_ncu.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"r02_{kernel}_ncu.json")) as f:
            return json.load(f)["traffic_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--obs", default="bits", choices=["bits", "u8", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-infer", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["strong", "weak"],
                    help="weak: the config's B segments per rank; strong: B split over the ranks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2011_12895_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    import paper_2011_12895_b200 as tlg

    obs_u8 = args.obs in ("u8", "bits") and cfg.obs_kind == "binary"
    obs_bits = obs_u8 and args.obs == "bits"
    T, D, A, hidden = cfg.unroll_len, cfg.obs_dim, cfg.n_actions, cfg.hidden
    if args.scaling == "strong" and cfg.batch_size % world:
        raise SystemExit(f"{cfg.batch_size} segments do not split over {world} ranks")
    S = cfg.batch_size // world if args.scaling == "strong" else cfg.batch_size

    def make_learner(S_):
        l_ = tlg.Learner("mlp", D, A, hidden, algo=cfg.algo, optimizer=cfg.optimizer,
                         max_segments=S_, unroll_len=T, device=local, obs_u8=obs_u8,
                         timing=False)
        l_.set_hyper(learning_rate=3e-4, batch_size=S_, unroll_len=T)
        l_.set_params(tlg.synth.init_params_f32(l_.n_params, 0.05,
                                                seed=cfg.seed).astype(np.float64))
        if world > 1:
            uid = [tlg.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            l_.comm_init(uid[0], world, rank)
        return l_
    lrn = make_learner(S)

    # distinct resident batches per rank, cycled so the inputs exceed L2 (126 MB): two
    # u8/f32 batches (obs >= 254 MB each) or four bit-packed ones (34 MB each at S=4096;
    # more batches at smaller per-rank shards, >= 136 MB resident per rank)
    def make_batches(S_):
        per = S_ * T * ((((D + 7) // 8 + 15) // 16 * 16 if obs_bits else
                         D * (1 if obs_u8 else 4)) + 17)  # + action/reward/blogp/value/done
        nb_ = max(4 if obs_bits else 2, -(-136_000_000 // per)) if obs_bits else 2
        host_ = [tlg.synth.make_segments(S_, T, D, A, seed=cfg.seed * 100 + rank * 10 + i,
                                         obs_kind=cfg.obs_kind, obs_u8=obs_u8)
                 for i in range(nb_)]
        if obs_bits:
            packed = []
            for h in host_:
                hb = h.slice(0, h.n_segments)
                hb.obs = tlg.synth.pack_bits(h.obs)
                packed.append(hb)
            # rows padded to 16-byte multiples in HBM: they feed the int8 GEMM's TMA directly
            pitch = ((D + 7) // 8 + 15) // 16 * 16
            dev_ = [tlg.DeviceSegmentBatch(h, local, bits=True, obs_dim=D, pitch=pitch)
                    for h in packed]
        else:
            dev_ = [tlg.DeviceSegmentBatch(h, local) for h in host_]
        return host_, dev_
    host, dev = make_batches(S)
    nb = len(dev)
    frames_per_step = [int(h.valid_steps.sum()) for h in host]
    resident_bytes = sum(sum(t.numel() * t.element_size() for t in d.t.values()) for d in dev)

    stream = torch.cuda.ExternalStream(lrn.stream(), device=local)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- device-resident timed region (no instrumentation: small steps replay as graphs)
    # (at least two passes over the resident batches: each one's CUDA graph is captured
    # on first use and replayed once before the timed region; at N > 1 at least 32 steps,
    # since the first timed region on a fresh multi-GPU box has read up to 1.7x slow)
    n_warm = max(args.warmup, 2 * nb, 32 if world > 1 else 0)
    for i in range(n_warm):
        lrn.train_step(dev[i % nb], on_device=True)
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    frames = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            lrn.train_step(dev[i % nb], on_device=True)
            frames += frames_per_step[i % nb]
            launches += lrn.last_launches()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_local = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_local)
    frames_all = sum_over_ranks(frames)
    value = frames_all / (ms_total / 1e3)
    ms_per_step = ms_total / args.steps

    # ---- at N>1: the other scaling mode's figure, measured in the same run
    other = None
    if world > 1:
        S_o = cfg.batch_size if args.scaling == "strong" else cfg.batch_size // world
        lw = make_learner(S_o)
        hw, dw = make_batches(S_o)
        fw = [int(h.valid_steps.sum()) for h in hw]
        for i in range(max(args.warmup, 2 * len(dw), 32)):
            lw.train_step(dw[i % len(dw)], on_device=True)
        sw = torch.cuda.ExternalStream(lw.stream(), device=local)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(sw)
        frw = 0
        for i in range(args.steps):
            lw.train_step(dw[i % len(dw)], on_device=True)
            frw += fw[i % len(dw)]
        e1.record(sw)
        torch.cuda.synchronize()
        msw = max_over_ranks(e0.elapsed_time(e1))
        other = {"value": sum_over_ranks(frw) / (msw / 1e3), "unit": "frames/s",
                 "segments_per_gpu": S_o, "global_batch_segments": S_o * world,
                 "ms_per_step": msw / args.steps}
        lw.close()
        del dw, hw
        torch.cuda.empty_cache()

    # ---- per-kernel CUDA-event times from separate instrumented (eager) steps
    lrn.set_timing(True)
    # every trunk GEMM: (kind, layer) -> CUDA-event ms per step
    gemms = [(k, l) for l in range(len(hidden)) for k in ("fwd", "dw", "dx")
             if not (k == "dx" and l == 0)]
    kern = {g: [] for g in gemms}
    kern["phases"] = []
    for i in range(max(5, args.steps // 2)):
        lrn.train_step(dev[i % nb], on_device=True)
        for g in gemms:
            kern[g].append(lrn.kernel_ms(*g))
        kern["phases"].append(lrn.phase_ms())
    lrn.set_timing(False)

    # ---- end to end through the C ABI with pinned host buffers: every step's batch is
    # copied H2D inside the timed region (pipelined: the copy of step k+1 overlaps step
    # k through tlg_learner_stage / tlg_learner_train_staged) and its statistics D2H'd.
    def pinned_view(h, bits=False, pitch=0):
        hb = h.slice(0, h.n_segments)
        if bits:
            hb.obs = tlg.synth.pack_bits(h.obs)
            if pitch:  # bit rows padded to `pitch` bytes on the host already
                padded = np.zeros(hb.obs.shape[:-1] + (pitch,), np.uint8)
                padded[..., :hb.obs.shape[-1]] = hb.obs
                hb.obs = padded
        pv = tlg.SegmentBatchView(hb, bits=bits, obs_dim=D)
        pv.pinned = []  # the pinned tensors must outlive the numpy views handed to the C ABI
        for k, a in pv.arrs.items():
            t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
            t.numpy()[...] = a
            pv.pinned.append(t)
            pv.arrs[k] = t.numpy()
        pv.c = tlg._capi.SegmentBatchC(
            h.n_segments, h.unroll_len, D, 2 if bits else (1 if obs_u8 else 0),
            *(pv.arrs[k].ctypes.data for k in ("obs", "action", "reward", "behavior_logp",
                                                 "value_est", "done", "bootstrap",
                                                 "valid_steps")), pitch)
        return pv

    def e2e_run(views):
        nsteps = max(10, args.steps)
        # warm the staged path: both staging slots allocated and graphs/maps built
        lrn.stage(views[0])
        lrn.stage(views[1])
        lrn.train_staged()
        lrn.train_staged()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fr = 0
        lrn.stage(views[0])
        for i in range(nsteps):
            # step i runs while batch i+1's H2D is issued (tlg_learner_train_staged_next)
            lrn.train_staged(views[(i + 1) % 2] if i + 1 < nsteps else None)
            fr += frames_per_step[i % 2]
        dt = max_over_ranks(time.perf_counter() - t0)
        return sum_over_ranks(fr) / dt

    # main e2e in the run's obs format; binary planes also reported as uint8 planes
    # bit rows padded to 16 B on the host (obs_pitch; +6 % bytes, no device re-pitch)
    host_pitch = ((D + 7) // 8 + 15) // 16 * 16 if obs_bits else 0
    pinned = [pinned_view(h, bits=obs_bits, pitch=host_pitch) for h in host[:2]]
    h2d = sum(a.nbytes for a in pinned[0].arrs.values())
    e2e_value = e2e_run(pinned)
    e2e_unpitched = None
    if obs_bits:  # dense ceil(D/8)-byte rows, re-pitched on the device
        pp = [pinned_view(h, bits=True) for h in host[:2]]
        e2e_unpitched = {"value": e2e_run(pp), "unit": "frames/s",
                         "h2d_bytes_per_step": sum(a.nbytes for a in pp[0].arrs.values()),
                         "d2h_bytes_per_step": 48 + 8,
                         "obs_format": "bit-packed planes, dense rows (re-pitched on device)"}

    # this box's pinned host->device bandwidth for the same bytes (PCIe; it bounds e2e)
    def h2d_gbs():
        src = torch.empty(h2d, dtype=torch.uint8, pin_memory=True)
        dst = torch.empty(h2d, dtype=torch.uint8, device=f"cuda:{local}")
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        return h2d * 5 / (time.perf_counter() - t0) / 1e9
    h2d_bw = h2d_gbs()
    e2e_alt = None
    if obs_bits:
        pu = [pinned_view(h) for h in host[:2]]
        e2e_alt = {"value": e2e_run(pu), "unit": "frames/s",
                   "h2d_bytes_per_step": sum(a.nbytes for a in pu[0].arrs.values()),
                   "d2h_bytes_per_step": 48 + 8, "obs_format": "uint8 planes"}

    # ---- device-resident replay: segments ingested once into HBM
    # slots, each step gathers a random draw of S slots on the device
    replay = None
    if obs_bits or not obs_u8:
        rep = tlg.Replay(lrn, 2 * S, bits=obs_bits)
        for k in range(2):  # (the first put also allocates the staging buffers)
            rep.put(np.arange(k * S, (k + 1) * S, dtype=np.uint32), pinned[k])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(2):
            rep.put(np.arange(k * S, (k + 1) * S, dtype=np.uint32), pinned[k])
        ingest_s = time.perf_counter() - t0
        rng = np.random.default_rng(rank)
        draws = [rng.permutation(2 * S)[:S].astype(np.uint32) for _ in range(args.steps + 2)]
        for i in range(2):
            rep.train_step(draws[i])
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fr = 0
        for i in range(args.steps):
            st = rep.train_step(draws[i + 2])
            fr += int(st[0]["n_samples"])
        dt = max_over_ranks(time.perf_counter() - t0)
        replay = {"value": sum_over_ranks(fr) / dt, "unit": "frames/s",
                  "ring_segments": 2 * S,
                  "ingest_gbs": 2 * h2d / ingest_s / 1e9,
                  "note": "tlg_learner_train_step_replay: random draws of S slots from a "
                          "2S-segment HBM ring (gathered on the device each step); ingest "
                          "= tlg_replay_put of two host batches"}
        rep.close()

    # ---- roofline of the dominant kernel (layer-1 forward GEMM)
    peaks, peak_src = measured_peaks()
    F = S * T
    dims = [D] + list(hidden)
    gflops = {(k, l): 2.0 * F * dims[l] * dims[l + 1] for (k, l) in gemms}
    gms = {g: float(np.mean(kern[g])) for g in gemms}
    flops_fwd1 = gflops[("fwd", 0)]
    t_fwd1 = gms[("fwd", 0)] / 1e3
    t_dw1 = gms[("dw", 0)] / 1e3
    # burst peak: the kernel is timed over a handful of instrumented steps, not a
    # seconds-long run (the sustained figure is reported beside it)
    peak = peaks.get("bf16_tflops", peaks.get("bf16_tflops_sustained"))
    ph = np.mean(np.array(kern["phases"]), axis=0)
    step_ms = float(ph[6])
    # the dominant kernel of the step: the trunk GEMM with the longest CUDA-event time
    dom_g = max(gemms, key=lambda g: gms[g])
    dom = {("fwd", 0): "fwd1", ("dw", 0): "dw1"}.get(dom_g, f"{dom_g[0]}{dom_g[1] + 1}")
    t_dom = gms[dom_g] / 1e3
    achieved = gflops[dom_g] / t_dom / 1e12
    desc = {
        "fwd1": ("gemm_i8_bits_fwd_dec_kernel layer-1 forward (tcgen05.mma kind::i8: "
                 "bit-packed binary planes x 3 fixed-point int8 weight pieces, exact int32 "
                 "accumulate; 256-column tiles, decoupled operand rings)"
                 if obs_bits else
                 "gemm_tf32x3_kernel layer-1 forward (tcgen05.mma kind::tf32, obs exact -> "
                 "2 MMA passes)"),
        "dw1": ("gemm_i8_bits_dw_kernel layer-1 dW = dZ1^T X (tcgen05.mma kind::i8: "
                "fixed-point dZ1 pieces x bit-packed planes, split-K)" if obs_bits else
                "gemm_tf32x3_kernel layer-1 dW = dZ1^T X (tcgen05.mma kind::tf32, MN-major "
                "operands, split-K)"),
    }.get(dom, f"gemm_tf32x3_kernel layer-{dom_g[1] + 1} {dom_g[0]} (tcgen05.mma kind::tf32, "
               f"3xTF32, {dims[dom_g[1]]}->{dims[dom_g[1] + 1]})")
    li, lo_ = dims[dom_g[1]], dims[dom_g[1] + 1]
    if dom == "fwd1":
        bytes_dom = F * D // (8 if obs_bits else 1) + 3 * hidden[0] * D + 2 * 4 * F * hidden[0]
    elif dom == "dw1":
        bytes_dom = 3 * F * hidden[0] + F * D // (8 if obs_bits else 1) + 4 * hidden[0] * D
    elif dom_g[0] == "fwd":
        bytes_dom = 8 * F * li + 8 * F * lo_ + 8 * li * lo_
    elif dom_g[0] == "dx":
        bytes_dom = 8 * F * lo_ + 4 * F * li + 8 * F * li + 8 * li * lo_
    else:
        bytes_dom = 8 * F * lo_ + 8 * F * li + 4 * li * lo_
    # the dominant kernel's own instruction ceiling (tools/mma_peak.cu: back-to-back
    # tcgen05.mma from smem on every SM pair, profiles/r02_mma_peak.json)
    try:
        with open(os.path.join(ROOT, "profiles", "r02_mma_peak.json")) as f:
            mp = json.load(f)
        if obs_bits and dom in ("fwd1", "dw1"):  # 3 kind::i8 MMAs per fp32-equivalent MAC
            own = {"kind": "tcgen05.mma kind::i8", "peak": mp["i8_tops"], "unit": "TOPS",
                   "achieved": 3 * achieved, "frac": 3 * achieved / mp["i8_tops"]}
        else:  # 3xTF32: 3 kind::tf32 MMAs per fp32 MAC (2 when one operand is exact)
            own = {"kind": "tcgen05.mma kind::tf32", "peak": mp["tf32_tflops"],
                   "unit": "TFLOP/s", "achieved": 3 * achieved,
                   "frac": 3 * achieved / mp["tf32_tflops"]}
        own["source"] = "profiles/r02_mma_peak.json"
    except Exception:
        own = None
    roofline = {
        "kernel": desc,
        "own_instruction_ceiling": own,
        "algorithmic_bytes_per_launch": bytes_dom,
        "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": _ncu_traffic(dom),
        "peak_source": f"{peak_src} bf16_tflops (burst, MEASURED_PEAKS.json)",
        "frac_of_sustained": achieved / peaks.get("bf16_tflops_sustained", peak),
        "algorithmic_flops_per_launch": gflops[dom_g],
        "ms_per_launch": t_dom * 1e3,
        "share_of_step": t_dom * 1e3 / step_ms,
        "note": "fp32-exact: 3xTF32 split (tf32 dense ceiling = half the bf16 peak, 2-3 MMA "
                "passes per K step) or exact int8 fixed point for binary planes",
    }
    kernels = {
        "fwd1_ms": t_fwd1 * 1e3, "dw1_ms": t_dw1 * 1e3,
        "dw1_tflops": 2.0 * F * hidden[0] * D / t_dw1 / 1e12,
        "phases_ms": {"stage": float(ph[0]), "fwd": float(ph[1]), "heads_returns_loss": float(ph[2]),
                      "bwd": float(ph[3]), "allreduce": float(ph[4]), "optimizer": float(ph[5]),
                      "step": step_ms},
    }
    kernels["gemm_ms"] = {f"{k}{l + 1}": gms[(k, l)] for (k, l) in gemms}
    total_flops = cfg.flops_per_frame() * F
    kernels["step_tflops"] = total_flops / (ms_per_step / 1e3) / 1e12

    # ---- InferenceServer batched forward (C4), replicas on every rank
    infer = None
    if not args.no_infer:
        c4 = CONFIGS["C4"]
        pol = tlg.Policy("mlp", c4.obs_dim, c4.n_actions, c4.hidden, device=local,
                         max_batch=c4.batch_size)
        n_p = (c4.obs_dim * c4.hidden[0] + c4.hidden[0] + c4.hidden[0] * c4.hidden[1] +
               c4.hidden[1] + (c4.n_actions + 1) * c4.hidden[1] + c4.n_actions + 1)
        pol.set_params(tlg.synth.init_params_f32(n_p, 0.05, seed=c4.seed).astype(np.float64))
        obs = tlg.synth.make_obs(c4.batch_size, c4.obs_dim, seed=c4.seed + rank)
        ob_t = torch.from_numpy(obs).cuda(local)
        lg_t = torch.empty(c4.batch_size, c4.n_actions, device=f"cuda:{local}")
        pr_t = torch.empty_like(lg_t)
        v_t = torch.empty(c4.batch_size, device=f"cuda:{local}")
        pstream = torch.cuda.ExternalStream(pol.stream(), device=local)
        for _ in range(3):
            pol.forward_device(ob_t, lg_t, pr_t, v_t)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(pstream)
        reps = max(5, args.steps)
        for _ in range(reps):
            pol.forward_device(ob_t, lg_t, pr_t, v_t)
        e1.record(pstream)
        torch.cuda.synchronize()
        ims = max_over_ranks(e0.elapsed_time(e1) / reps)
        # pinned host buffers on both sides (kept alive while their views are used)
        obs_pin_t = torch.from_numpy(obs).pin_memory()
        obs_pin = obs_pin_t.numpy()
        outs_t = [torch.empty(c4.batch_size, c4.n_actions, pin_memory=True),
                  torch.empty(c4.batch_size, c4.n_actions, pin_memory=True),
                  torch.empty(c4.batch_size, pin_memory=True)]
        outs = tuple(t.numpy() for t in outs_t)
        pol.forward(obs_pin, out=outs)
        barrier()
        t0 = time.perf_counter()
        for _ in range(10):
            pol.forward(obs_pin, out=outs)
        idt_sync = max_over_ranks((time.perf_counter() - t0) / 10)
        # pipelined stream of batches (tlg_policy_forward_async): batch k+1's H2D and batch
        # k-1's D2H overlap batch k's forward; each batch's results are waited for
        obs_pins = [obs_pin, torch.from_numpy(obs.copy()).pin_memory().numpy()]
        outs2 = [outs, tuple(torch.empty_like(t, pin_memory=True).numpy() for t in outs_t)]
        tk = [pol.forward_async(obs_pins[0], outs2[0])]
        pol.wait(tk[0])
        barrier()
        reps_p = 20
        t0 = time.perf_counter()
        tk = []
        for k in range(reps_p):
            tk.append(pol.forward_async(obs_pins[k % 2], outs2[k % 2]))
            if k >= 1:
                pol.wait(tk[k - 1])
        pol.wait(tk[-1])
        idt = max_over_ranks((time.perf_counter() - t0) / reps_p)
        infer = {"metric": "InferenceServer actions/sec", "config": c4.name, "note": c4.note,
                 "value": world * c4.batch_size / (ims / 1e3), "unit": "actions/s",
                 "ms_per_batch": ims,
                 "tflops": 2.2426e6 * c4.batch_size / (ims / 1e3) / 1e12,
                 "e2e": {"value": world * c4.batch_size / idt, "unit": "actions/s",
                         "h2d_bytes_per_batch": obs.nbytes,
                         "d2h_bytes_per_batch": c4.batch_size * (2 * c4.n_actions + 1) * 4,
                         "note": "pinned host batches through tlg_policy_forward_async, two in "
                                 "flight (H2D / forward / D2H overlapped), every batch waited for",
                         "synchronous": world * c4.batch_size / idt_sync}}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            fps, cores, sample, _ = reference_cpu(cfg, seconds=10.0)
            cpu = {"value": fps, "unit": "frames/s", "cores": cores, "kind": "reference",
                   "sample": sample}
        except Exception as e:
            cpu = {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}
        # the reference learner at num_shards = 1 too, and the same MLP on the
        # CPU (the fp64 oracle port; the reference cannot run an MLP)
        others = []
        try:
            fps1, c1, sample1, _ = reference_cpu(cfg, seconds=5.0, shards=1)
            others.append({"value": fps1, "unit": "frames/s", "cores": c1, "kind": "reference",
                           "sample": sample1})
        except Exception as e:
            others.append({"value": None, "kind": "reference", "sample": f"unavailable: {e}"})
        try:
            others.append(oracle_mlp_cpu(cfg))
        except Exception as e:
            others.append({"value": None, "kind": "port", "sample": f"unavailable: {e}"})
        cpu["others"] = others
        if infer is not None:
            try:
                infer["cpu_baseline"] = oracle_policy_cpu(CONFIGS["C4"])
            except Exception as e:
                infer["cpu_baseline"] = {"value": None, "kind": "port", "sample": f"unavailable: {e}"}

    # ---- the drop-in C++ learner::Learner (reference-facing API) at C3, N=1
    dropin = None
    exe = os.path.join(ROOT, "integration", "_build", "dropin_bench")
    if rank == 0 and world == 1 and cfg.name == "C3" and os.path.exists(exe):
        try:
            out = subprocess.run([exe, str(cfg.batch_size), "3"], capture_output=True, text=True,
                                 timeout=300)
            dropin = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, not raised
            dropin = {"unavailable": f"{type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "warmup_steps_run": n_warm,
            "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "note": cfg.note, "algo": cfg.algo,
                       "optimizer": cfg.optimizer, "obs_dim": D, "hidden": list(hidden),
                       "n_actions": A, "unroll_len": T, "segments_per_gpu": S,
                       "global_batch_segments": S * world,
                       "frames_per_gpu_step": F,
                       "obs_format": ("bit-packed binary planes (rows padded to 16 B in HBM)"
                                      if obs_bits else "u8 planes" if obs_u8 else "f32"),
                       "parallelism": f"dp{world}",
                       "gemm_precision": ("layer 1 exact int8 fixed point (binary planes), "
                                          "other GEMMs 3xTF32 (fp32-exact)" if obs_bits else
                                          "3xTF32 (fp32-exact)"),
                       "l2": f"inputs > L2: {nb} resident batches cycled, "
                             f"{resident_bytes / 1e6:.0f} MB in total"},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 48 + 8, "h2d_gbs_measured": h2d_bw,
                    "note": "pinned host SoA batch H2D each step (same obs format as value; "
                            "bit rows padded to 16 B), pipelined one step ahead on a copy "
                            "stream; stats D2H each step"},
            ("weak_scaling" if args.scaling == "strong" else "strong_scaling"): other,
            "dropin_e2e": dropin,
            "e2e_alt_format": e2e_alt,
            "e2e_dense_rows": e2e_unpitched,
            "device_replay": replay,
            "gpu_launches": launches,
            "roofline": roofline,
            "kernels": kernels,
            "infserver": infer,
            "cpu_baseline": cpu,
            "clocks": clk.result(),
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
