#!/usr/bin/env python
"""Benchmark of the SWR / Block Two-Pass hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config layer4k|L8k|L16k|L32k|L4k_b16|paper_d16|layer4k_f32|tiny] [--op swr|mix]
                    [--path auto|ffma|tc]

A step is one pass of the whole hot path over one batch of synthetic input:
SWR forward (swr_fwd) + backward (swr_bwd) -- or, with --op mix, the Phalanx
mixer forward + backward -- on inputs already resident in HBM.  Metric
(BASELINE.json): fwd+bwd tokens/s, plus achieved HBM GB/s of the dominant
kernel against the measured copy peak (MEASURED_PEAKS.json).

Timing: W untimed warm-up steps; then K steps back to back, each bracketed by
CUDA events on the launching stream; barrier + synchronize around the loop;
per-rank sum of step times, max over ranks.  When a step's inputs exceed 2x the
L2 (every graded config) nothing is flushed between steps, so every dirty line a
step leaves in L2 is written back inside the next step's events (no deferred
write-back goes unpaid).  Smaller inputs get an L2 flush between steps (write a
2x-L2 buffer, then read another); the flushed timing of the large configs is
reported beside the headline as "l2_flushed".  Multi-GPU (torchrun): layer4k
and the other single-GPU configs run the same per-GPU workload on every rank
(batch x head sharding, no collective; weak scaling); `bxh` splits BASELINE
configs[3]'s B = 64 over the ranks (strong scaling); `sp131k` shards L.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, L, H, D, dtype)
    "layer4k": (8, 4096, 16, 128, "bf16"),    # BJ configs[1]: the metric's workload
    "L8k": (8, 8192, 16, 128, "bf16"),        # BJ configs[2]: 64K tokens/GPU
    "L16k": (4, 16384, 16, 128, "bf16"),
    "L32k": (2, 32768, 16, 128, "bf16"),
    "L4k_b16": (16, 4096, 16, 128, "bf16"),
    "bxh": (64, 8192, 16, 128, "bf16"),       # BJ configs[3]: B = 64 split over the ranks
    "paper_d16": (8, 8192, 128, 16, "bf16"),  # the paper's head shape d=16, h=128
    "layer4k_f32": (8, 4096, 16, 128, "f32"),  # BJ configs[1] shape with fp32 storage (FFMA path)
    "tiny": (1, 64, 1, 16, "f32"),            # BJ configs[0]
    "sp131k": (1, 131072, 16, 128, "bf16"),   # BJ configs[4]: sequence-parallel across ranks
}
SP_CONFIGS = {"sp131k"}
SPLIT_CONFIGS = {"bxh"}  # global batch split over the ranks (strong scaling)
EXTRA = ("L8k", "L16k", "L32k")  # BJ configs[2] lines measured beside the default workload
METRIC = "SWR fwd+bwd tokens/s and achieved HBM GB/s vs B200 peak at 4K-32K, 1/2/4/8 GPUs"


def esize(dt):
    return 2 if dt == "bf16" else 4


LAYER_GROUPS = 8  # --op layer: q and k shared by 8 groups of heads


def algo_bytes(op, B, L, H, D, dt):
    """Algorithmic HBM bytes per launch; halo re-reads excluded."""
    e, n = esize(dt), B * L * H
    if op == "swr":
        return {"fwd": n * (2 * D + 1) * e, "bwd": n * (3 * D + 2) * e}
    if op == "layer":  # q, zk are [B, L, G, D]: read once per group, dq / dzk written per group
        nt, G = B * L, min(LAYER_GROUPS, H)
        return {"fwd": nt * (2 * G * D + 2 * H * D + H) * e, "bwd": nt * (4 * G * D + 3 * H * D + 2 * H) * e}
    return {"fwd": n * (4 * D + 1) * e, "bwd": n * (7 * D + 2) * e}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index, period=0.001):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm: the fp64 oracle on the host cores
# ---------------------------------------------------------------------------
def oracle_step_fn(op, inp_host, rows, threads=0):
    import oracle
    from swr_inputs import to64
    sl = slice(0, rows)
    h = {k: to64(v[sl]) for k, v in inp_host.items()}
    if op == "swr":
        def step():
            oracle.swr_fwd(h["u"], h["a"], threads=threads)
            oracle.swr_bwd(h["u"], h["a"], h["G"], threads=threads)
    elif op == "layer":
        def step():
            oracle.layer_mix_fwd(h["q"], h["zk"], h["v"], h["za"], threads=threads)
            oracle.layer_mix_bwd(h["q"], h["zk"], h["v"], h["za"], h["dy"], threads=threads)
    else:
        def step():
            oracle.mix_fwd(h["q"], h["k"], h["v"], h["a"], threads=threads)
            oracle.mix_bwd(h["q"], h["k"], h["v"], h["a"], h["dy"], threads=threads)
    return step


def make_host_inputs(op, B, L, H, D, dt, seed):
    import torch
    from swr_inputs import layer_inputs, mix_inputs, swr_inputs
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    if op == "layer":
        G = min(LAYER_GROUPS, H)
        return layer_inputs(B, L, H, D, G, G, dtype=dtype, seed=seed)
    f = swr_inputs if op == "swr" else mix_inputs
    return f(B, L, H, D, dtype=dtype, seed=seed)


def cpu_baseline(op, inp_host, B, L, H, budget_s=10.0):
    """The oracle as it stands on a bounded sample of the workload: enough batch rows
    that its (b, h) thread pool can occupy every host core, repeated until
    `budget_s` of wall time; then the same with one thread on one row."""
    import math

    import oracle
    host = os.cpu_count() or 1
    rows = max(1, min(B, math.ceil(host / H)))

    def timed(rows_, threads, budget):
        step = oracle_step_fn(op, inp_host, rows_, threads)
        step()  # build + first touch
        n, t0 = 0, time.perf_counter()
        while True:
            step()
            n += 1
            el = time.perf_counter() - t0
            if el >= budget or n >= 1000:
                break
        return rows_ * L * n / el, n, el, oracle.oracle.last_threads

    v, n, el, used = timed(rows, 0, budget_s)
    v1, n1, el1, _ = timed(1, 1, budget_s / 2)
    return {"value": v, "unit": "tokens/s", "cores": used, "host_cores": host,
            "kind": "oracle", "value_1thread": v1,
            "sample": f"{rows} of {B} batch rows (all {H} heads, full length) fwd+bwd, {n} repetitions "
                      f"in {el:.1f} s on {used} threads (one per (b, h) pair, at most the host's {host} "
                      f"cores); 1 thread: 1 row, {n1} repetitions in {el1:.1f} s; fp64 C oracle"}


def run_reference(args, cfg_name, B, L, H, D, dt):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inp = make_host_inputs(args.op, 1, L, H, D, dt, seed=1)
    import oracle
    step = oracle_step_fn(args.op, inp, 1)
    for _ in range(args.warmup):
        step()
    t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        t.append(time.perf_counter() - t0)
    sec = sum(t) / len(t)
    val = L / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if (cfg_name in SP_CONFIGS or cfg_name in SPLIT_CONFIGS) else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg_name, "B": B, "L": L, "H": H, "d_head": D, "op": args.op,
                   "sample_rows_per_step": 1},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": oracle.oracle.last_threads,
                         "host_cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"1 of {B} batch rows (all {H} heads, L={L}) fwd+bwd per step"},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def step_fns(P, op, g):
    """fwd() and bwd() of one step of the hot path on device-resident inputs g."""
    if op == "swr":
        return (lambda: P.swr_fwd(g["u"], g["a"])), (lambda: P.swr_bwd(g["u"], g["a"], g["G"]))
    if op == "layer":  # sigma on the logits, 8 groups for q and k
        return ((lambda: P.phalanx_layer_mix(g["q"], g["zk"], g["v"], g["za"])),
                (lambda: P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])))
    return ((lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"])),
            (lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="layer4k", choices=sorted(CONFIGS))
    ap.add_argument("--op", default="swr", choices=["swr", "mix", "layer"])
    ap.add_argument("--path", default="auto", choices=["auto", "ffma", "tc"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the L8k/L16k/L32k lines")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="batch-row chunks of the e2e copy pipeline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    B, L, H, D, dt = CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, args.config, B, L, H, D, dt)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # SWR_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo -- a functional check of the
        # multi-rank harness (max over ranks, batch split, SP halo) on a one-GPU box; the
        # ranks then share the GPU, so its numbers are not scaling measurements
        one_gpu = os.environ.get("SWR_BENCH_ONE_GPU") == "1"
        local = 0 if one_gpu else local
        torch.cuda.set_device(local)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2512_13921_b200 as P
    P.set_path({"auto": P.SWR_PATH_AUTO, "ffma": P.SWR_PATH_FFMA, "tc": P.SWR_PATH_TC}[args.path])

    sp = args.config in SP_CONFIGS
    if sp:
        # sequence parallel: one L-shard per rank (multiples of 16), carrier halo over NCCL
        from paper_2512_13921_b200 import dist as sdist
        if args.op != "swr":
            raise SystemExit("sequence-parallel bench supports --op swr")
        full = make_host_inputs("swr", B, L, H, D, dt, seed=3)
        lens = sdist.sp_shard_lengths(L, world)
        lo = sum(lens[:rank])
        inp_host = {k: (v[:, lo:lo + lens[rank]].contiguous() if v.dim() >= 3 else v)
                    for k, v in full.items()}
        Ls = lens[rank]
        grp = dist.group.WORLD if world > 1 else None
    else:
        if args.config in SPLIT_CONFIGS:
            # BJ configs[3]: the global batch split into contiguous per-rank slices
            if B % world:
                raise SystemExit(f"--config {args.config}: B={B} does not split over {world} ranks")
            B = B // world
        # per-rank shard of the batch (batch x head sharding): seed by global batch offset
        inp_host = make_host_inputs(args.op, B, L, H, D, dt, seed=1 + 1000 * rank)
        Ls = L
    g = {k: v.to(dev) for k, v in inp_host.items()}
    stream = torch.cuda.current_stream()

    if sp and world > 1:
        state = {}

        def fwd():
            x, state["cin"] = sdist.swr_sp_fwd(g["u"], g["a"], group=grp)
            return x

        def bwd():
            return sdist.swr_sp_bwd(g["u"], g["a"], g["G"], carry_in=state.get("cin"), group=grp)
    else:
        fwd, bwd = step_fns(P, args.op, g)

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_rd = torch.zeros_like(flush)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    def l2_flush():
        # write > 2x L2, then read another > 2x L2 buffer: the write evicts every line
        # of the previous step, the read pushes the flush's own dirty lines back to HBM,
        # so the step starts with a clean L2 holding nothing it will read (the state
        # ncu's --cache-control all gives a kernel) and pays no stray write-back
        flush.zero_()
        flush_sink.copy_(flush_rd.sum())

    def in_bytes(gg):
        return sum(v.numel() * v.element_size() for v in gg.values())

    def timed(fwd_, bwd_, steps, warmup, flushed):
        """(total ms of `steps` steps, per-step fwd ms, per-step bwd ms), CUDA events.
        Back to back unless `flushed`.  The GPU is first given ~2 ms of sleep so the
        host enqueues ahead of it and no launch latency lands inside the events.  The
        total comes from two events around the loop; a second loop with an event
        between fwd and bwd of every step gives the split."""
        for _ in range(warmup):
            if flushed:
                l2_flush()
            fwd_()
            bwd_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        head_start = 4_000_000  # SM cycles (~2 ms): lets the host run ahead of the GPU
        if flushed:  # per-step events; the flush between steps stays outside them
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
            torch.cuda._sleep(head_start)
            n0 = P.launch_count()
            for s_ in range(steps):
                l2_flush()
                ev[s_][0].record(stream)
                fwd_()
                ev[s_][1].record(stream)
                bwd_()
                ev[s_][2].record(stream)
            timed.launches = P.launch_count() - n0
            torch.cuda.synchronize()
            tf = [e[0].elapsed_time(e[1]) for e in ev]
            tb = [e[1].elapsed_time(e[2]) for e in ev]
            return sum(tf) + sum(tb), tf, tb
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(head_start)
        n0 = P.launch_count()
        e0.record(stream)
        for _ in range(steps):
            fwd_()
            bwd_()
        e1.record(stream)
        timed.launches = P.launch_count() - n0
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        torch.cuda._sleep(head_start)
        for s_ in range(steps):
            ev[s_][0].record(stream)
            fwd_()
            ev[s_][1].record(stream)
            bwd_()
            ev[s_][2].record(stream)
        torch.cuda.synchronize()
        return total, [e[0].elapsed_time(e[1]) for e in ev], [e[1].elapsed_time(e[2]) for e in ev]

    red_dev = dev if world == 1 or dist.get_backend() == "nccl" else torch.device("cpu")

    def max_over_ranks(x):
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    b2b = in_bytes(g) > 2 * l2  # inputs larger than L2: no flush between steps
    copies0 = P.layout_copies()
    with ClockSampler(dev.index if world == 1 else local) as clk:
        t_total, t_fwd, t_bwd = timed(fwd, bwd, args.steps, args.warmup, flushed=not b2b)
    launches = timed.launches  # our kernels launched inside the timed loop
    assert P.layout_copies() == copies0, "operands were copied inside the timed region"
    if world > 1:
        dist.barrier()
    ms_per_step = max_over_ranks(t_total) / args.steps
    tokens_per_step = B * L if sp else B * L * world
    value = tokens_per_step / (ms_per_step / 1e3)

    bytes_ = algo_bytes(args.op, B, Ls, H, D, dt)
    # the split loop's event between the two kernels stops the backward's early start
    # (programmatic dependent launch), so its fwd / bwd times add up to more than a
    # step: attribute the step time to the two kernels in the split loop's proportion
    sf, sb = statistics.mean(t_fwd), statistics.mean(t_bwd)
    step_ms = ms_per_step
    mf, mb = step_ms * sf / (sf + sb), step_ms * sb / (sf + sb)
    dom = "bwd" if mb >= mf else "fwd"
    peak, peak_kind = load_peaks()
    ach = bytes_[dom] / (mb if dom == "bwd" else mf) / 1e6  # GB/s
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f)
        rec = tr.get(f"{args.op}_{dom}_{args.config}_{dt}")
        if isinstance(rec, dict):
            traffic, traffic_src = rec.get("bytes"), rec.get("source")

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if (sp or args.config in SPLIT_CONFIGS) else "weak", "vs_baseline": None,
        "dtype": dt, "data": "synthetic",
        "config": {"workload": args.config, "B": B * (world if args.config in SPLIT_CONFIGS else 1),
                   "B_per_rank": B, "L": L, "H": H, "d_head": D, "op": args.op,
                   "global_batch": B if sp else B * world, "seq_len": L,
                   "parallelism": (f"sp{world} (sequence shards, one-block carrier halo via "
                                   f"{(dist.get_backend().upper() + ' send/recv') if world > 1 else 'none'})") if sp else
                                  f"dp{world} (batch x head shards, no collective)",
                   "timing": ("back to back, no L2 flush: inputs "
                              f"{in_bytes(g) >> 20} MiB > 2x L2 ({l2 >> 20} MiB), so each step pays the "
                              "previous step's deferred write-back") if b2b else
                             (f"L2 flushed between steps ({flush.numel() * 4 >> 20} MiB write + "
                              f"{flush_rd.numel() * 4 >> 20} MiB read, outside the events)"),
                   "path": args.path, "last_path": {0: "none", 1: "ffma", 2: "tc"}[P.last_path()]},
        "fwd_ms": mf, "bwd_ms": mb,
        "split_note": ("fwd_ms / bwd_ms: the step time split in the proportion of a second loop with an "
                       "event between the two kernels of each step (split loop: fwd %.4f ms, bwd %.4f ms)" % (sf, sb)),
        "hbm_gbs": {"fwd": bytes_["fwd"] / mf / 1e6, "bwd": bytes_["bwd"] / mb / 1e6,
                    "fwd_bwd": (bytes_["fwd"] + bytes_["bwd"]) / (mf + mb) / 1e6},
        "roofline": {"bound": "hbm", "kernel": f"{args.op}_{dom}", "achieved": ach, "peak": peak,
                     "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                     "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "traffic_source": traffic_src or "not captured for this workload",
                     "algorithmic_bytes": bytes_[dom]},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if b2b:
        # the same steps with the L2 flushed between them (each step's deferred
        # write-back is then paid by the flush, outside the events)
        f_tot, f_fwd, f_bwd = timed(fwd, bwd, min(args.steps, 20), 3, flushed=True)
        fm = max_over_ranks(f_tot) / len(f_fwd)
        line["l2_flushed"] = {"value": tokens_per_step / (fm / 1e3), "ms_per_step": fm,
                              "fwd_ms": statistics.mean(f_fwd), "bwd_ms": statistics.mean(f_bwd)}
    if (args.config == "layer4k" and not sp and not args.no_extra):
        # BJ configs[2]: 64K tokens per GPU at L = 8K / 16K / 32K, same op and timing
        line["workloads"] = {}
        for name in EXTRA:
            Bx, Lx, Hx, Dx, dtx = CONFIGS[name]
            gx = {k: v.to(dev) for k, v in make_host_inputs(args.op, Bx, Lx, Hx, Dx, dtx, seed=2 + 1000 * rank).items()}
            fx, bx = step_fns(P, args.op, gx)
            bx_ = in_bytes(gx) > 2 * l2
            x_tot, x_fwd, x_bwd = timed(fx, bx, min(args.steps, 20), 3, flushed=not bx_)
            xm = max_over_ranks(x_tot) / len(x_fwd)
            xb = algo_bytes(args.op, Bx, Lx, Hx, Dx, dtx)
            line["workloads"][name] = {
                "B": Bx, "L": Lx, "value": Bx * Lx * world / (xm / 1e3), "unit": "tokens/s", "ms_per_step": xm,
                "fwd_ms": xm * statistics.mean(x_fwd) / (statistics.mean(x_fwd) + statistics.mean(x_bwd)),
                "bwd_ms": xm * statistics.mean(x_bwd) / (statistics.mean(x_fwd) + statistics.mean(x_bwd)),
                "hbm_gbs_fwd_bwd": (xb["fwd"] + xb["bwd"]) / xm / 1e6,
                "timing": "back to back" if bx_ else "L2 flushed"}
            del gx
    torch.cuda.synchronize()

    # end to end through the public API with host buffers (pinned), copies timed.
    # Batch rows are independent, so the step is pipelined over row chunks on three
    # streams: host->device copy of chunk c+1 and device->host copy of chunk c-1
    # overlap the kernels of chunk c (PCIe is full duplex; the copies dominate).
    if not args.no_e2e and not (sp and world > 1):
        pin = {k: v.pin_memory() for k, v in inp_host.items()}
        ne = min(args.steps, 10)
        h2d = sum(v.numel() * v.element_size() for v in pin.values())
        nch = min(B, args.e2e_chunks) if not sp else 1
        rows = [(B * c // nch, B * (c + 1) // nch) for c in range(nch)]
        s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

        def chunk_step(r0, r1):
            c = {k: (v[r0:r1] if v.dim() >= 3 else v) for k, v in g.items()}
            if args.op == "swr":
                du, da, _ = P.swr_bwd(c["u"], c["a"], c["G"])
                return (P.swr_fwd(c["u"], c["a"]), du, da)
            if args.op == "layer":
                dq, dzk, dv, dza, _ = P.phalanx_layer_mix_bwd(c["q"], c["zk"], c["v"], c["za"], c["dy"])
                return (P.phalanx_layer_mix(c["q"], c["zk"], c["v"], c["za"]), dq, dzk, dv, dza)
            dq, dk, dv, da, _ = P.phalanx_mix_bwd(c["q"], c["k"], c["v"], c["a"], c["dy"])
            return (P.phalanx_mix(c["q"], c["k"], c["v"], c["a"]), dq, dk, dv, da)

        outs_host = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        for s in range(ne + 2):
            l2_flush()
            torch.cuda.synchronize()
            e0.record(stream)
            for st_ in (s_in, s_c, s_out):
                st_.wait_event(e0)
            done = []
            for ci, (r0, r1) in enumerate(rows):
                with torch.cuda.stream(s_in):
                    for k, v in pin.items():
                        if v.dim() >= 3:
                            g[k][r0:r1].copy_(v[r0:r1], non_blocking=True)
                        elif ci == 0:
                            g[k].copy_(v, non_blocking=True)
                    ev_in = torch.cuda.Event()
                    ev_in.record(s_in)
                s_c.wait_event(ev_in)
                with torch.cuda.stream(s_c):
                    outs = chunk_step(r0, r1)
                    ev_c = torch.cuda.Event()
                    ev_c.record(s_c)
                if outs_host is None:
                    outs_host = [[torch.empty((rr1 - rr0,) + tuple(o.shape[1:]), dtype=o.dtype, pin_memory=True)
                                  for o in outs] for rr0, rr1 in rows]
                s_out.wait_event(ev_c)
                with torch.cuda.stream(s_out):
                    for o, oh in zip(outs, outs_host[ci]):
                        oh.copy_(o, non_blocking=True)
                done.append(outs)  # keep the chunk's device outputs alive until the copies ran
            stream.wait_stream(s_out)
            e1.record(stream)
            torch.cuda.synchronize()
            if s >= 2:
                times.append(e0.elapsed_time(e1))
        d2h = sum(o.numel() * o.element_size() for oc in outs_host for o in oc)
        te = torch.tensor([sum(times) / len(times)], device=red_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": tokens_per_step / (te.item() / 1e3), "unit": "tokens/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": te.item(), "steps": ne, "pipeline_chunks": nch}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.op, inp_host, B, Ls, H)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
