#!/usr/bin/env python
"""Benchmark of the numerical-entanglement hot path on B200 (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
M=3 streams of N=2^24 int32 samples in [-2^11, 2^11-1], one 256-tap filter,
geometry derive_params(3, 64) = (l=21, k=21); full linear convolution of every
entangled stream, all 3 outputs recovered (failed=None pivots on stream 0 and
checks the redundant stream).  One step = one launch of the fused
entangle -> conv -> extract kernel over the whole batch, inputs resident in HBM.
The kernel is the exact digit-sliced tensor-core convolution on the 5th-gen
tensor cores (tcgen05.mma kind::i8, TMEM accumulators, warp-specialised): the
35-bit entangled words become 5 int8 digit planes, the 12-bit taps 2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1 (torchrun): halo-split weak scaling -- rank p owns a 2^24-sample slice of
an N*2^24-sample signal; the K-1 = 255-sample halo comes from rank p-1 over
NCCL once at setup; the timed region has no collective.  Rank 0 prints one
JSON line.  --impl reference times the reference algorithm's CPU restatement
(oracle/, all host threads) on the same workload; only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "entangled int conv output samples/s; overhead vs non-entangled conv (%)"
UNIT = "samples/s"
WORKLOAD = "cfg2: M=3, N=2^24 int32 in [-2^11,2^11), K=256 taps, (m,w,l,k)=(3,64,21,21), full conv"
B2B_ROUNDS = 3  # alternations of the back-to-back entangled / plain blocks (overhead headline)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other-config section")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work for the cpu_baseline sample")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every
    ~2 ms while the timed region runs (the same counters nvidia-smi's
    clocks.sm / clocks_event_reasons.* report); nvidia-smi is the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self.source = "nvml"
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            masks = [(nm, getattr(N, attr)) for nm, attr in self.REASONS if hasattr(N, attr)]

            def poll():
                while not self._stop.is_set():
                    self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for nm, mask in masks:
                        if bits & mask:
                            self.reasons.add(nm)
                    time.sleep(self.period)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            time.sleep(3 * self.period)
        except Exception as exc:  # NVML unavailable: one nvidia-smi read instead
            self.source = f"nvidia-smi ({type(exc).__name__})"
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=1)
            return
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=10).stdout.split(",")
            self.samples, self.max_mhz = [int(float(out[0]))], int(float(out[1]))
        except Exception:
            pass

    def summary(self) -> dict:
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": self.source,
                "sm_mhz_min": min(sm) if sm else None}


# -------------------------------------------------------------- workload --

def make_inputs(rank: int, n: int, K: int):
    """Rank 0 holds the canonical cfg2 draw (seed 2); rank p > 0 draws its
    slice from seed (2, p) -- same shapes and value distribution."""
    from paper_1509_03838_b200 import workloads

    wl0 = workloads.make(2, n=n, K=K)  # the filter is drawn after the streams: full draw
    if rank == 0:
        return wl0.params, wl0.c, wl0.g
    rng = np.random.default_rng([2, rank])
    c = rng.integers(-(1 << 11), 1 << 11, (3, n), dtype=np.int64)
    return wl0.params, c, wl0.g  # every rank uses the same filter


def event_time(fn, stream, reps=1):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    return a, b


# ------------------------------------------------------------ our device path --

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1509_03838_b200 import _device as D
    from paper_1509_03838_b200 import fused
    from paper_1509_03838_b200._lib import (BENCH_IMMA, BENCH_TC05, MAC_F64, MAC_G64, MAC_I32, MAC_NAMES, MAC_S64,
                                            MAC_W64, imma_flavor, is_imma)
    from paper_1509_03838_b200.hostpath import ChunkedEntangledConv

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # NENT_BENCH_BACKEND=gloo exercises the N>1 path when fewer GPUs than ranks
    # exist (exchange through host memory; ranks share devices round-robin)
    backend = os.environ.get("NENT_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    xdev = dev if backend == "nccl" else torch.device("cpu")  # where collectives' tensors live

    n, K = 1 << 24, 256
    params, c_np, g = make_inputs(rank, n, K)
    m, H = params.m, K - 1
    c_dev = torch.from_numpy(c_np).to(dev).to(torch.int32)
    if world > 1:  # halo-split: the samples left of this rank's slice come from rank-1
        Hp = (H + 3) // 4 * 4  # K-1 rounded up to 4 words: the kernel's tiles then start 16-byte aligned
        halo = torch.zeros((m, Hp), dtype=torch.int32, device=xdev)
        ops = []
        if rank + 1 < world:
            ops.append(dist.P2POp(dist.isend, c_dev[:, n - Hp:].contiguous().to(xdev), rank + 1))
        if rank > 0:
            ops.append(dist.P2POp(dist.irecv, halo, rank - 1))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        x_dev = torch.cat([halo.to(dev), c_dev], dim=1).contiguous()
        n_out = n + (H if rank == world - 1 else 0)  # the last rank also owns the K-1 tail
        period, n_in, y_begin = Hp + n + H, Hp + n, Hp  # rank 0 keeps a zero halo (left edge)
    else:
        x_dev = c_dev
        n_out, period, n_in, y_begin = n + H, n + H, n, 0

    max_c = 1 << 11
    eps_bound = max_c * ((1 << params.l) + 1)
    flavor = fused.conv_flavor(eps_bound, g, n_out=n_out)             # imma5x2 for cfg2
    core_flavor = fused.conv_flavor(eps_bound, g, allow_imma=False)   # f64: the CUDA-core path
    plain_same = flavor                                               # same kernel, same digits
    plain_fast = fused.conv_flavor(max_c, g, n_out=n_out)             # fastest plain: imma2x2
    plain_core = fused.conv_flavor(max_c, g, allow_imma=False)        # i32
    taps = {f: D.taps_tensor(g, f) for f in {flavor, core_flavor, plain_same, plain_fast, plain_core}}
    # IMMA: digit-split Toeplitz tap tables prepared once (the taps are fixed)
    tables = {f: D.imma_table(taps[f], K, f, y_begin) for f in taps}
    # output rows at 128-byte aligned starts (a padded row pitch; the kernels take
    # one pointer per row), so every warp's 128-byte store is one whole line
    pitch = (n_out + 31) // 32 * 32
    d_dev = torch.empty((m, pitch), dtype=torch.int32, device=dev)[:, :n_out]
    y_plain = torch.empty((m, pitch), dtype=torch.int32, device=dev)[:, :n_out]
    mismatch = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def fused_step(fl=flavor):
        D.fused_conv(x_dev, taps[fl], K, params.l, fl, None, params.w > 32, period, n_in=n_in,
                     y_begin=y_begin, n_out=n_out, out=d_dev, mismatch=mismatch,
                     imma_table=tables[fl])

    def failed_step(r=1, fl=flavor):  # one stream lost: recovery from the two survivors
        D.fused_conv(x_dev, taps[fl], K, params.l, fl, r, params.w > 32, period, n_in=n_in,
                     y_begin=y_begin, n_out=n_out, out=d_dev, imma_table=tables[fl])

    def plain(fl):
        D.conv(x_dev, taps[fl], K, fl, period=period, y_begin=y_begin, n_out=n_out, out=y_plain,
               imma_table=tables[fl])

    for _ in range(args.warmup):
        fused_step()
        plain(plain_same)
        plain(plain_fast)
    torch.cuda.synchronize(dev)

    exact = None
    known = None
    if rank == 0 and world == 1:  # parity of the benchmarked output itself
        known = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())["cfg2"]["d"]
        exact = sha(d_dev.to(torch.int64).cpu().numpy()) == known and int(mismatch.item()) == 0

    # ---------------- timed region: exactly K steps ----------------
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        ev0, ev1 = event_time(fused_step, stream, args.steps)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=xdev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / args.steps
    samples_job = m * n_out if world == 1 else m * (n * world + H)
    value = samples_job / (ms_step / 1e3)
    if world > 1:  # parity of every shard against one single-GPU run over the whole signal
        exact = check_shards(D, d_dev, rank, world, n, K, params, g, flavor, dev, xdev)

    # ---------------- the plain convolutions timed like `value` ----------------
    # K back-to-back launches each on the same stream, CUDA events around them
    # (the same protocol as the timed region above), the three blocks alternated
    # B2B_ROUNDS times and each candidate's median taken, so the entangled and
    # the plain blocks see the same box state (one plain block alone varied
    # 0.117-0.136 ms between boxes while the entangled one stayed at 0.146-0.149)
    rounds = {"entangled": [], "plain_same_kernel": [], "plain_fastest": []}
    blocks = (("entangled", fused_step), ("plain_same_kernel", lambda: plain(plain_same)),
              ("plain_fastest", lambda: plain(plain_fast)))
    for _ in range(B2B_ROUNDS):
        for name, fn in blocks:
            fn()
            torch.cuda.synchronize(dev)
            a0, a1 = event_time(fn, stream, args.steps)
            torch.cuda.synchronize(dev)
            rounds[name].append(a0.elapsed_time(a1) / args.steps)
    b2b = {k: float(np.median(v)) for k, v in rounds.items()}

    # ---------------- interleaved comparisons (per-launch CUDA events) ----------------
    cands = {
        "entangled": lambda: fused_step(flavor),
        "entangled_cuda_core": lambda: fused_step(core_flavor),
        "entangled_failed_r1": lambda: failed_step(1),
        "plain_same_kernel": lambda: plain(plain_same),
        "plain_fastest": lambda: plain(plain_fast),
        "plain_cuda_core_same_width": lambda: plain(core_flavor),
        "plain_cuda_core_narrowest": lambda: plain(plain_core),
    }
    evs = {k: [] for k in cands}
    for _ in range(max(5, min(args.steps, 11))):
        for k, fn in cands.items():
            evs[k].append(event_time(fn, stream))
    torch.cuda.synchronize(dev)
    t = {k: [a.elapsed_time(b) for a, b in v] for k, v in evs.items()}
    med = {k: statistics.median(v) for k, v in t.items()}

    def ovh(a, b):
        return statistics.median([(x - y) / y * 100 for x, y in zip(t[a], t[b])])

    # ---------------- measured pipe peaks (roofline denominators) ----------------
    peaks = {}
    for kind in (BENCH_TC05, BENCH_IMMA, MAC_F64, MAC_I32, MAC_W64, MAC_S64, MAC_G64):
        grid = 148 if kind == BENCH_TC05 else 148 * 8
        iters = {BENCH_TC05: 2000, BENCH_IMMA: 1024}.get(kind, 4096)
        D.microbench(kind, grid, 256, 64)
        best = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            macs = D.microbench(kind, grid, 256, iters)
            b.record(stream)
            torch.cuda.synchronize(dev)
            best = max(best, macs / (a.elapsed_time(b) / 1e3))
        peaks[MAC_NAMES[kind]] = best
    np_, ng = (flavor >> 8) & 15, (flavor >> 12) & 15
    # the dominant kernel's average launch duration over the timed region (one
    # fused launch per step, back to back on `stream`); the interleaved
    # per-launch median is reported beside it
    kern_ms = ms_step
    macs_alg = m * n * K                      # M*N*K
    digit_macs = macs_alg * np_ * ng          # int8 digit products the method needs
    achieved = 2 * digit_macs / (kern_ms / 1e3) / 1e12
    kernel_kind = D.imma_kernel(flavor, K, m, True)
    peak_key = "tcgen05_i8" if kernel_kind == "tcgen05" else "imma_s8_mma_sync"
    peak = 2 * peaks[peak_key] / 1e12
    kt = (K + 127 + 127) // 128 * 128      # tcgen05 Toeplitz band: K + 127 padded to 128
    issued_macs = m * (n + K - 1) * kt * np_ * ng if kernel_kind == "tcgen05" else None
    traffic = None
    tf = REPO / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(MAC_NAMES[flavor], {}).get("bytes_per_launch")
        except Exception:
            traffic = None

    # ---------------- e2e through the host-buffer path ----------------
    # Every rank pushes its own host-resident input ([halo | slice] for N > 1)
    # through the pipeline; the job time is the max over ranks.
    e2e = None
    if world == 1:
        xin_np = c_np.astype(np.int32)
    else:
        xin_np = x_dev.cpu().numpy()  # this rank's staged [halo | slice] words
    n_e = xin_np.shape[1]
    pipe = ChunkedEntangledConv(params, n_e, g, flavor)  # 2^20-sample chunks, output lag 1
    c_host = torch.from_numpy(xin_np).pin_memory()
    d_host = torch.empty((m, n_e + H), dtype=torch.int32).pin_memory()
    o0 = 0 if world == 1 else y_begin  # this rank's outputs inside the pipeline's full conv

    def shard_ok() -> bool:
        return bool(torch.equal(d_host[:, o0:o0 + n_out], d_dev.cpu()))

    pipe.capture(c_host, d_host)  # the whole multi-stream job as one CUDA graph
    d_host.zero_()
    pipe.replay()
    torch.cuda.synchronize(dev)
    ok = shard_ok()
    reps = max(3, min(args.steps, 8))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        pipe.replay()
        torch.cuda.synchronize(dev)
    single_s = (time.perf_counter() - t0) / reps
    # streaming: `reps` steps as one continuous pipeline (each step still
    # copies all its inputs in and all its outputs out; fill/drain once)
    pipe.capture(c_host, d_host, jobs=reps)
    d_host.zero_()
    pipe.replay()
    torch.cuda.synchronize(dev)
    ok = ok and shard_ok()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    pipe.replay()
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / reps
    tt = torch.tensor([e2e_s, single_s, 0.0 if ok else 1.0], dtype=torch.float64, device=xdev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s, single_s, bad = (float(v) for v in tt.tolist())
    if exact is not None:
        exact = exact and bad == 0.0
    e2e = {"value": samples_job / e2e_s, "unit": UNIT, "h2d_bytes_per_step": pipe.h2d_bytes() * world,
           "d2h_bytes_per_step": pipe.d2h_bytes() * world, "ms_per_step": e2e_s * 1e3,
           "steps_streamed": reps, "single_step_ms": single_s * 1e3, "bit_exact_vs_device_output": bad == 0.0,
           "path": "ChunkedEntangledConv on every rank: pinned int32 host -> 3-stage pipeline (H2D stream / "
                   "fused-kernel stream / D2H stream, 2^20-sample chunks each moved as one 2-D DMA "
                   "per direction, D2H lagging H2D by one chunk, 4-buffer ring, 256-byte-aligned "
                   "host transfers), "
                   "the steps captured as one continuous CUDA graph (a stream of batches: the next "
                   "step's input copies overlap the previous step's last output copies); wall clock "
                   "over all steps incl. sync, max over ranks; single_step_ms = one step per graph "
                   "replay + sync" + ("; N > 1: each rank's host input is its [halo | slice]" if world > 1 else ""),
           "pcie_floor_ms": "~4.0 per GPU (201 MB each way at the ~50 GB/s measured concurrently)",
           "kernels_per_step": pipe.launches // reps}

    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = other_configs(D, fused, dev, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c_np, g, params, args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 digits x int8 digits -> int32 -> int64 (exact integer; int32 in/out)",
            "data": "synthetic (canonical seeded cfg2 draw, SURVEY.md 8d)",
            "config": {"workload": WORKLOAD, "samples_per_step": samples_job,
                       "parallelism": "halo-split" if world > 1 else "single GPU",
                       "l2": "inputs 201 MB + outputs 201 MB per step > 126 MB L2; no flush needed",
                       "mac_flavor": MAC_NAMES[flavor], "failed": None, "verify_redundant_stream": True},
            "overhead_pct": (b2b["entangled"] - b2b["plain_same_kernel"]) / b2b["plain_same_kernel"] * 100,
            "overhead": {
                "headline": "back-to-back: K launches of the fused entangled kernel vs K launches of the "
                            "same kernel and digit geometry on the plain streams, the blocks alternated "
                            f"{B2B_ROUNDS} times, median per candidate",
                "back_to_back_ms": b2b, "back_to_back_rounds_ms": rounds,
                "back_to_back_vs_plain_fastest_pct": (b2b["entangled"] - b2b["plain_fastest"])
                                                     / b2b["plain_fastest"] * 100,
                "interleaved_vs_plain_same_kernel_pct": ovh("entangled", "plain_same_kernel"),
                "vs_plain_same_kernel_pct": ovh("entangled", "plain_same_kernel"),
                "vs_plain_fastest_pct": ovh("entangled", "plain_fastest"),
                "cuda_core_entangled_vs_plain_same_width_pct": ovh("entangled_cuda_core",
                                                                   "plain_cuda_core_same_width"),
                "vs_plain_cuda_core_narrowest_pct": ovh("entangled", "plain_cuda_core_narrowest"),
                "flavors": {"entangled": MAC_NAMES[flavor], "entangled_cuda_core": MAC_NAMES[core_flavor],
                            "plain_same_kernel": MAC_NAMES[plain_same], "plain_fastest": MAC_NAMES[plain_fast],
                            "plain_cuda_core_narrowest": MAC_NAMES[plain_core]},
                "ms": med,
                "note": "plain_same_kernel runs the identical kernel/digit geometry on the plain streams "
                        "(isolates entangle+extract); plain_fastest uses the digits the 12-bit plain "
                        "samples need (2 planes instead of the entangled words' 5); entangled_failed_r1 "
                        "loses stream 1: the two survivors are convolved and all three outputs recovered "
                        "(the lost stream is never computed)"},
            "roofline": {"bound": "tensor",
                         "pipe": ("tcgen05.mma kind::i8 (5th-gen tensor cores, TMEM accumulators)"
                                  if kernel_kind == "tcgen05" else "IMMA (mma.sync m16n8k32 s8)"),
                         "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": (f"nent::tcc::conv_tc05_kernel<true,{np_},{kt // 32}> ({MAC_NAMES[flavor]})"
                                    if kernel_kind == "tcgen05"
                                    else f"nent::conv_imma_kernel<3,{ng},true> ({MAC_NAMES[flavor]})"),
                         "algorithmic_per_launch": {"conv_macs": macs_alg, "digit_macs": digit_macs,
                                                    "digit_planes": np_, "tap_digits": ng,
                                                    "tensor_macs_issued": issued_macs,
                                                    "note": "achieved counts the method's digit MACs "
                                                            "(M*N*K*np*ng); the tcgen05 Toeplitz band "
                                                            "issues KT/K more (zero taps outside the band)"},
                         "issued_tops": (2 * issued_macs / (kern_ms / 1e3) / 1e12) if issued_macs else None,
                         "launch_ms": {"timed_region_avg": kern_ms, "interleaved_median": med["entangled"]},
                         "peak_source": (f"measured in this run: nent_microbench {peak_key} "
                                         + ("(tcgen05.mma 128x128x32 chains, 1 CTA/SM)" if kernel_kind == "tcgen05"
                                            else "(16 independent accumulators per warp, 148*8 CTAs x 8 warps)")),
                         "cuda_core_path": {"flavor": MAC_NAMES[core_flavor],
                                            "achieved_tflops": 2 * macs_alg / (med["entangled_cuda_core"] / 1e3) / 1e12,
                                            "peak_tflops": 2 * peaks[MAC_NAMES[core_flavor]] / 1e12},
                         "peaks_measured_gmac_s": {k: v / 1e9 for k, v in peaks.items()},
                         # BASELINE.json north_star's roofline: the 64-bit integer multiply rate
                         # of the CUDA cores (measured here: IMAD.WIDE and generic 64-bit MAC
                         # chains); the fused kernel's exact int64 conv MACs (M*N*K) per second
                         # against it
                         "int64_cuda_core_roofline": {
                             "conv_macs_per_s": macs_alg / (kern_ms / 1e3),
                             "peak_w64_macs_per_s": peaks["w64"], "peak_g64_macs_per_s": peaks["g64"],
                             "frac_vs_w64": macs_alg / (kern_ms / 1e3) / peaks["w64"],
                             "frac_vs_g64": macs_alg / (kern_ms / 1e3) / peaks["g64"],
                             "note": "the tensor-core digit slicing delivers exact 64-bit convolution "
                                     "MACs faster than the CUDA cores can issue 64-bit multiplies"}},
            "e2e": e2e,
            "gpu_launches": args.steps,  # one fused kernel per step (tap table prepared before)
            "exact": exact,
            "mismatches": int(mismatch.item()),
            "clocks": clocks.summary(),
            "other_configs": extras,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def check_shards(D, d_dev, rank, world, n, K, params, g, flavor, dev, xdev):
    """Halo-split parity: every rank hashes its recovered output slice; rank 0
    regenerates all slices' inputs, convolves the concatenated signal in one
    single-GPU fused launch and compares slice by slice."""
    import torch
    import torch.distributed as dist

    mine = np.frombuffer(bytes.fromhex(sha(d_dev.to(torch.int64).cpu().numpy())), dtype=np.uint8)
    hashes = [torch.zeros(32, dtype=torch.uint8, device=xdev) for _ in range(world)]
    dist.all_gather(hashes, torch.from_numpy(mine.copy()).to(xdev))
    if rank != 0:
        return None
    H = K - 1
    full = np.concatenate([make_inputs(p, n, K)[1] for p in range(world)], axis=1)
    x = torch.from_numpy(full).to(dev).to(torch.int32)
    L = full.shape[1] + H
    out = torch.empty((params.m, L), dtype=torch.int32, device=dev)
    gd = D.taps_tensor(g, flavor)
    D.fused_conv(x, gd, K, params.l, flavor, None, True, L, n_in=full.shape[1], out=out)
    ok = True
    for p in range(world):
        a, b = p * n, (p + 1) * n + (H if p == world - 1 else 0)
        want = sha(out[:, a:b].to(torch.int64).cpu().numpy())
        good = want == bytes(hashes[p].cpu().numpy()).hex()
        if not good:
            print(f"shard {p}: digest mismatch (mine {bytes(hashes[p].cpu().numpy()).hex()[:16]}, "
                  f"want {want[:16]}; local {sha(d_dev.to(torch.int64).cpu().numpy())[:16] if p == 0 else ''})",
                  file=sys.stderr)
            if p == 0:
                dd = d_dev.to(torch.int64).cpu().numpy()
                ww = out[:, a:b].to(torch.int64).cpu().numpy()
                bad = np.argwhere(dd != ww)
                print(f"shard 0: {len(bad)} differing samples, first {bad[:4].tolist()}, "
                      f"shapes {dd.shape} {ww.shape}", file=sys.stderr)
        ok = ok and good
    return ok


def other_configs(D, fused, dev, stream):
    """The other BASELINE configs through the same fused path: ms per launch,
    output samples/s, and the known-answer digest check (no failure)."""
    import torch

    from paper_1509_03838_b200 import workloads
    from paper_1509_03838_b200._lib import MAC_NAMES

    digests = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())
    res = {}
    for cfg in (1, 3, 5):
        wl = workloads.make(cfg)
        p = wl.params
        c = torch.from_numpy(wl.c).to(dev).to(torch.int32)
        n, K = wl.n, wl.K
        L = n + K - 1
        out = torch.empty((wl.m, L), dtype=torch.int32, device=dev)
        mm = torch.zeros(1, dtype=torch.int64, device=dev)
        xb = int(np.abs(wl.c).max()) * ((1 << p.l) + 1)
        chain = wl.scale is not None
        if chain:  # entangle -> scale -> add -> perm as interleave + gather, then conv + extract
            a = torch.from_numpy(wl.add).to(dev)
            add = D.shift_add(a, a, p.l)
            perm = torch.from_numpy(wl.perm).to(dev).to(torch.int32)  # prepared once, like the taps
            xb = xb * abs(wl.scale) + int(add.abs().max())
            ct = torch.empty((n, wl.m), dtype=torch.int32, device=dev)
            xg = torch.empty((wl.m, n), dtype=torch.int32, device=dev)
        fl = fused.conv_flavor(xb, wl.g, n_out=L)
        gd = D.taps_tensor(wl.g, fl)
        tab = D.imma_table(gd, K, fl, 0)
        # m > 3 chain: tcgen05 conv of the chain rows + verifying extract (the
        # route fused.entangled_chain_conv takes), else the fused kernel
        split = (chain and D.imma_kernel(fl, K, wl.m, True) != "tcgen05"
                 and D.imma_kernel(fl, K, wl.m, False) == "tcgen05")
        if split:
            delta = torch.empty((wl.m, L), dtype=torch.int32, device=dev)

        def run():
            if chain:
                # chain words in the coalesced interleave pass, then one record gather
                D.interleave_chain(c, p.l, wl.scale, add, out=ct)
                D.gather_records(ct, perm, out=xg)
                if split:
                    D.conv(xg, gd, K, fl, period=L, n_out=L, out=delta)
                    D.extract_verify(delta, wl.m, p.l, 0, p.w > 32, mm, out=out)
                else:
                    D.fused_conv(xg, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm,
                                 pre_entangled=True, imma_table=tab)
            else:
                D.fused_conv(c, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm,
                             imma_table=tab)

        for _ in range(3):
            run()
        torch.cuda.synchronize(dev)
        ok = sha(out.to(torch.int64).cpu().numpy()) == digests[f"cfg{cfg}"]["d"] and int(mm.item()) == 0
        reps = 20 if cfg == 1 else 5
        a, b = event_time(run, stream, reps)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        res[f"cfg{cfg}"] = {"flavor": MAC_NAMES[fl], "ms": ms,
                            "kernel": (("tcgen05 conv + verifying extract" if split else D.imma_kernel(fl, K, wl.m, True))
                                       if (fl & 0xFF) == 7 else "cuda-core"), "samples_per_s": wl.m * L / (ms / 1e3),
                            "conv_gmac_s": wl.m * n * K / (ms / 1e3) / 1e9, "exact": ok}
    # cfg4 inner products (65,536 x 4,096 per stream, 3 streams)
    wl = workloads.make(4)
    c = torch.from_numpy(wl.c).to(dev).to(torch.int32)
    r = fused.entangled_inner(wl.params, c, wl.g)  # public API once: digest + redundant check
    ok = sha(r.outputs.data.to(torch.int64).cpu().numpy()) == digests["cfg4_inner"]["d"] and r.mismatches == 0
    from paper_1509_03838_b200._lib import MAC_G64
    gd = D.taps_tensor(wl.g, MAC_G64)
    outd = torch.empty((3, c.shape[1]), dtype=torch.int64, device=dev)

    def inner():
        D.fused_inner(c, gd, wl.params.l, None, True, MAC_G64, out_dtype=torch.int64)

    inner()
    a, b = event_time(inner, stream, 5)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / 5
    res["cfg4_inner"] = {"flavor": r.flavor, "ms": ms, "hbm_gb_s": c.numel() * 4 / (ms / 1e3) / 1e9,
                         "hbm_frac_of_measured": c.numel() * 4 / (ms / 1e3) / 1e9 / 6540.5, "exact": ok}
    del outd
    del c
    torch.cuda.empty_cache()
    return res


# -------------------------------------------------- stream per GPU (cfg3/cfg5) --

def device_barrier(dev, backend, group=None):
    """Cross-rank ordering of device work: with NCCL a one-element all-reduce
    on the current stream (every rank's earlier kernels complete before any
    rank's later ones run; no host sync); with gloo (ranks sharing one GPU in
    the CPU-side tests) a device sync plus a host barrier."""
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        dist.all_reduce(torch.zeros(1, device=dev), group=group)
    else:
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)


def run_stream_per_gpu(cfg: int, steps: int, warmup: int, dev, backend: str) -> dict | None:
    """BASELINE cfg3 (M=4) / cfg5 (M=8) with one entangled stream per GPU
    (reference pipeline.py:90-137): rank i holds c_i; one step
    = ring shift of c_{i-1} (P2P), the worker's fused entangle [-> scale ->
    add -> permute] -> conv kernel giving delta_i, the drop of rank
    r = step mod M (every GPU fails in turn), and the position-sharded K3 on
    every survivor reading its slice of the other survivors' deltas straight
    from their HBM (CUDA IPC peer pointers over NVLink).  Reported: recovered
    output samples/s of the job (max over ranks), the plain per-GPU
    convolution (no entanglement, no recovery) timed the same way, the
    recovery alone, and the reference digest of the recovered outputs for
    every dropped rank (gathered to rank 0)."""
    import torch
    import torch.distributed as dist

    from paper_1509_03838_b200 import _device as D
    from paper_1509_03838_b200 import workloads
    from paper_1509_03838_b200._lib import MAC_NAMES
    from paper_1509_03838_b200.distributed import PeerRows, StreamPerGPU
    from paper_1509_03838_b200.fused import chain_operands, conv_flavor

    rank, world = dist.get_rank(), dist.get_world_size()
    wl = workloads.make(cfg)
    p, m, n, K = wl.params, wl.m, wl.n, wl.K
    if world != m:
        return None
    L = n + K - 1
    drv = StreamPerGPU(p)
    c_own = torch.from_numpy(wl.c[rank].copy()).to(dev).to(torch.int32)
    chain = wl.scale is not None
    add_ent = perm = None
    xb = int(np.abs(wl.c).max()) * ((1 << p.l) + 1)
    if chain:
        add_dev, perm = chain_operands(wl.add, wl.perm, n)
        add_ent = D.shift_add(add_dev.to(torch.int32), add_dev.to(torch.int32), p.l, out_dtype=torch.int32)
        xb = xb * abs(wl.scale) + int(np.abs(wl.add).max()) * ((1 << p.l) + 1)
    flavor = conv_flavor(xb, wl.g, n_out=L, gather=chain)
    plain_flavor = conv_flavor(int(np.abs(wl.c).max()) * (abs(wl.scale) if chain else 1)
                               + (int(np.abs(wl.add).max()) if chain else 0), wl.g, n_out=L, gather=chain)
    g_dev = D.taps_tensor(wl.g, flavor)
    gp_dev = D.taps_tensor(wl.g, plain_flavor)
    tab = D.imma_table(g_dev, K, flavor, 0)
    ptab = D.imma_table(gp_dev, K, plain_flavor, 0)
    sum_g = int(np.abs(wl.g).sum())
    ddt = torch.int32 if xb * sum_g < (1 << 31) else torch.int64
    delta = torch.empty((L,), dtype=ddt, device=dev)
    y_plain = torch.empty((1, L), dtype=torch.int32, device=dev)
    add_plain = torch.from_numpy(wl.add).to(dev).to(torch.int32) if chain else None
    # the survivors' rows, mapped once (the buffer is persistent across steps)
    rows = PeerRows(drv, delta)
    width = -(-L // (m - 1))
    d_out = torch.empty((m, width), dtype=torch.int32, device=dev)

    def worker():
        prev = drv.ring_shift(c_own)
        D.chain_conv(prev, c_own, g_dev, K, p.l, flavor, L, n_in=n, scale=wl.scale or 1, add=add_ent,
                     perm=perm, out=delta, imma_table=tab)

    def recover(failed):
        mb, me = rows.bounds(failed)
        if me > mb:
            rows.extract(failed, out=d_out[:, : me - mb])

    def step(s):
        worker()
        device_barrier(dev, backend)   # every delta complete before any peer read
        recover(s % m)
        device_barrier(dev, backend)   # every read done before the next step rewrites delta

    def plain():
        D.chain_conv(None, c_own, gp_dev, K, p.l, plain_flavor, L, n_in=n, scale=wl.scale or 1,
                     add=add_plain, perm=perm, out=y_plain[0], imma_table=ptab)

    stream = torch.cuda.current_stream(dev)

    def timed(fn, k):
        device_barrier(dev, backend)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(k):
            fn(i)
        b.record(stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([a.elapsed_time(b) / k], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(warmup):
        step(i)
        plain()
    ms_ent = timed(step, steps)
    ms_plain = timed(lambda i: plain(), steps)
    worker()
    device_barrier(dev, backend)
    ms_rec = timed(lambda i: recover(i % m), steps)
    ms_worker = timed(lambda i: worker(), steps)
    device_barrier(dev, backend)
    # parity: the recovered outputs of every dropped rank against the reference digest
    want = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())[f"cfg{cfg}"]["d"]
    exact = {}
    for r in list(range(m)) + [None]:
        d, mb, me = rows.extract(r)
        full = drv.gather(d, L, r, dst=0)
        if rank == 0:
            exact[str(r)] = sha(full.to(torch.int64).cpu().numpy()) == want
        del full, d
    rows.close()
    samples = m * L
    return {"workload": f"cfg{cfg}: M={m} streams of N={n}, K={K}, (m,w,l,k)=({p.m},{p.w},{p.l},{p.k})"
                        + (f", chain scale {wl.scale} -> add -> perm -> conv" if chain else ", full conv"),
            "parallelism": f"stream-per-GPU ({m} ranks, one entangled stream each)",
            "ms_per_step": ms_ent, "value": samples / (ms_ent / 1e3), "unit": UNIT,
            "plain_ms_per_step": ms_plain, "plain_value": samples / (ms_plain / 1e3),
            "overhead_pct": (ms_ent - ms_plain) / ms_plain * 100,
            "worker_ms": ms_worker, "recovery_ms": ms_rec,
            "recovery_note": "K3 on each survivor's 1/(M-1) slice reading the other survivors' deltas in place "
                             "(CUDA IPC peer pointers), dropped rank = step mod M",
            "flavor": MAC_NAMES[flavor], "plain_flavor": MAC_NAMES[plain_flavor],
            "exact_every_dropped_rank": exact if rank == 0 else None,
            "backend": backend}


# ------------------------------------------------------------- CPU baseline --

def cpu_pipeline_time(O, c: np.ndarray, g: np.ndarray, params, threads: int = 0):
    """Reference algorithm on the CPU: entangle -> full conv on the entangled
    streams -> recover all 3 (failed=None); then the plain conv."""
    K = len(g)
    t0 = time.perf_counter()
    pad = np.zeros((c.shape[0], c.shape[1] + K - 1), dtype=np.int64)
    pad[:, : c.shape[1]] = c
    eps = O.entangle(pad, params.l, threads)
    delta = O.circ_conv(eps, g, threads, wide=False)
    d = O.disentangle(delta, params.m, params.l, params.w, None, threads)
    t_ent = time.perf_counter() - t0
    t0 = time.perf_counter()
    y = O.circ_conv(pad, g, threads, wide=False)
    t_plain = time.perf_counter() - t0
    assert np.array_equal(d, y)
    return t_ent, t_plain, d.shape[0] * d.shape[1]


def host_desc():
    import platform
    model = ""
    try:
        model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                      if ln.startswith("model name")), "")
    except OSError:
        pass
    return f"{model} ({os.cpu_count()} logical CPUs, {platform.machine()})"


def host_threads() -> int:
    """Every host thread this process may run on (torchrun exports
    OMP_NUM_THREADS=1 for N > 1, which would otherwise cap the OpenMP team)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(c, g, params, target_s: float):
    from oracle import oracle as O

    threads = host_threads()
    ns = 1 << 16
    t, _, _ = cpu_pipeline_time(O, c[:, :ns], g, params, threads)
    ns = int(min(c.shape[1], max(ns, ns * target_s / 2 / max(t, 1e-6))))
    t_ent, t_plain, samples = cpu_pipeline_time(O, c[:, :ns], g, params, threads)
    return {"value": samples / t_ent, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {ns} samples of each of the 3 cfg2 streams, K=256, full conv "
                      f"(entangle + conv + recover), oracle/nent_oracle.c OpenMP",
            "plain_value": samples / t_plain, "overhead_pct": (t_ent - t_plain) / t_plain * 100,
            "seconds": t_ent + t_plain, "host": host_desc()}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # only rank 0 runs the CPU reference arm
    from oracle import oracle as O

    params, c, g = make_inputs(0, 1 << 24, 256)
    threads = host_threads()
    ns = 1 << 16  # bounded sample per step, sized so the run stays within a few minutes
    t, _, _ = cpu_pipeline_time(O, c[:, :ns], g, params, threads)
    budget = 150.0 / max(args.steps + args.warmup, 1)
    ns = int(min(c.shape[1], max(ns, ns * budget / 2 / max(t, 1e-6))))
    for _ in range(args.warmup):
        cpu_pipeline_time(O, c[:, :ns], g, params, threads)
    te, tp = [], []
    for _ in range(args.steps):
        a, b, samples = cpu_pipeline_time(O, c[:, :ns], g, params, threads)
        te.append(a)
        tp.append(b)
    t_step = sum(te) / len(te)
    value = samples / t_step
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64 (reference numpy semantics)",
        "data": "synthetic (canonical seeded cfg2 draw, SURVEY.md 8d)",
        "config": {"workload": WORKLOAD, "sample": f"first {ns} samples per stream"},
        "impl": "reference",
        "overhead_pct": statistics.median([(a - b) / b * 100 for a, b in zip(te, tp)]),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"first {ns} samples of each cfg2 stream per step (K=256, full "
                                   f"conv, entangle+conv+recover), oracle/nent_oracle.c OpenMP",
                         "host": host_desc()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
