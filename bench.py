#!/usr/bin/env python
"""Benchmark of the numerical-entanglement hot path on B200 (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
M=3 streams of N=2^24 int32 samples in [-2^11, 2^11-1], one 256-tap filter,
full linear convolution of every entangled stream, all 3 outputs recovered
(failed=None pivots on stream 0 and checks the redundant stream).  One step =
one launch of the fused entangle -> conv -> extract kernel over the whole
batch, inputs resident in HBM.  The codec geometry is derive_params(3, 48) =
(l=16, k=16) by default (--w 64 selects the (21, 21) geometry; the recovered
outputs are identical): its 28-bit entangled words are 4
int8 digit planes on the 5th-gen tensor cores (tcgen05.mma kind::i8, TMEM
accumulators), the fused m = 3 kernel conv_tc05_m3.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                  [--w 48|64] [--config 2|3|5]

N>1 (torchrun): cfg2 halo-split weak scaling through distributed.HaloSplit --
rank p owns a 2^24-sample slice; the halo comes from rank p-1 over NCCL once
at setup; the timed region has no collective.  At N=4 and N=8 the
stream-per-GPU configs (cfg3 on 4 GPUs, cfg5 on 8) are measured as well and
attached as "stream_per_gpu"; --config 3|5 makes them the headline line.
--impl reference times the reference algorithm's CPU restatement (oracle/,
all host threads) on the same workload; only rank 0 runs it.
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
B2B_ROUNDS = 3  # alternations of the back-to-back entangled / plain blocks (overhead headline)
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--w", type=int, default=48, choices=[48, 64],
                    help="codec word width of the cfg2 geometry: 48 -> (3,48,16,16), 64 -> (3,64,21,21)")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 5],
                    help="2: cfg2 (halo-split for N>1); 3/5: stream-per-GPU cfg3 (N=4) / cfg5 (N=8)")
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


def compact(o):
    """Floats to 6 significant digits (the line stays a few KB)."""
    if isinstance(o, float):
        return float(f"{o:.6g}")
    if isinstance(o, dict):
        return {k: compact(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [compact(v) for v in o]
    return o


def hbm_peak() -> tuple[float, str]:
    """Measured HBM copy bandwidth (GB/s) of this pool's B200s."""
    try:
        v = float(json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def workload_name(w: int) -> str:
    from paper_1509_03838_b200.params import derive_params
    p = derive_params(3, w)
    return (f"cfg2: M=3, N=2^24 int32 in [-2^11,2^11), K=256 taps, (m,w,l,k)=({p.m},{p.w},{p.l},{p.k}), "
            "full conv, failed=None + redundant-stream check")


def bench_config(world: int, w: int, cfg: int = 2) -> dict:
    """The `config` object both arms print (identical dicts)."""
    if cfg != 2:
        return {"workload": f"cfg{cfg} stream-per-GPU", "parallelism": "stream-per-GPU", "n_ranks": world}
    return {"workload": workload_name(w), "samples_per_step": 3 * ((1 << 24) * world + 255),
            "parallelism": "halo-split" if world > 1 else "single GPU",
            "l2": "inputs 201 MB + outputs 201 MB per GPU and step > 126 MB L2; no flush needed"}


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
        self.power_w: list[float] = []
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
                    try:
                        self.power_w.append(N.nvmlDeviceGetPowerUsage(h) / 1e3)
                    except Exception:
                        pass
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
                "sm_mhz_min": min(sm) if sm else None,
                # NVML's board power over the same samples (its averaging window is longer than
                # the timed region: run for seconds the headline kernel sits at the 1,000 W limit
                # with sw_power_cap set)
                "power_w_max": max(self.power_w) if self.power_w else None}


# -------------------------------------------------------------- workload --

def make_inputs(rank: int, n: int, K: int, w: int = 48):
    """Rank 0 holds the canonical cfg2 draw (seed 2); rank p > 0 draws its
    slice from seed (2, p) -- same shapes and value distribution."""
    from paper_1509_03838_b200 import workloads
    from paper_1509_03838_b200.params import derive_params

    wl0 = workloads.make(2, n=n, K=K)  # the filter is drawn after the streams: full draw
    p = derive_params(3, w)
    if rank == 0:
        return p, wl0.c, wl0.g
    rng = np.random.default_rng([2, rank])
    c = rng.integers(-(1 << 11), 1 << 11, (3, n), dtype=np.int64)
    return p, c, wl0.g  # every rank uses the same filter


def event_time(fn, stream, reps=1):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    return a, b


def timed_ms(fn, stream, reps: int) -> float:
    """Average ms per call of `reps` back-to-back calls (CUDA events on `stream`)."""
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = event_time(fn, stream, reps)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


# ------------------------------------------------------------ our device path --

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1509_03838_b200 import _device as D
    from paper_1509_03838_b200 import fused
    from paper_1509_03838_b200._lib import BENCH_IMMA, BENCH_TC05, MAC_F64, MAC_NAMES, imma_flavor
    from paper_1509_03838_b200.distributed import HaloSplit
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

    if args.config in (3, 5):  # stream-per-GPU as the headline line
        res = run_stream_per_gpu(args.config, args.steps, args.warmup, dev, backend)
        if rank == 0:
            if res is None:
                print(json.dumps({"metric": METRIC, "unavailable": f"cfg{args.config} needs WORLD_SIZE == "
                                  f"{4 if args.config == 3 else 8} (one stream per GPU), got {world}"}))
            else:
                print(json.dumps({"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
                                  "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                                  "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                                  "overhead_pct": res["overhead_pct"], "dtype": "int32 in/out, exact int64",
                                  "data": "synthetic (canonical seeded draw, SURVEY.md 8d)",
                                  "config": bench_config(world, args.w, args.config), "stream_per_gpu": res,
                                  "gpu_launches": None}))
        if world > 1:
            dist.destroy_process_group()
        return

    n, K = 1 << 24, 256
    params, c_np, g = make_inputs(rank, n, K, args.w)
    m, H = params.m, K - 1
    c_dev = torch.from_numpy(c_np).to(dev).to(torch.int32)
    if world > 1:  # halo-split: [halo | slice] from rank-1, once, outside the timed region
        halo_drv = HaloSplit(params, K)
        x_dev = halo_drv.exchange_halo(c_dev)
        win = halo_drv.window(n)
    else:
        x_dev = c_dev
        win = {"period": n + H, "n_in": n, "y_begin": 0, "n_out": n + H}
    n_out, period, n_in, y_begin = win["n_out"], win["period"], win["n_in"], win["y_begin"]

    max_c = 1 << 11
    eps_bound = max_c * ((1 << params.l) + 1)
    flavor = fused.conv_flavor(eps_bound, g, n_out=n_out)             # imma4x2 (w=48) / imma5x2 (w=64)
    core_flavor = fused.conv_flavor(eps_bound, g, allow_imma=False)   # f64: the CUDA-core path
    plain_same = flavor                                               # same kernel, same digits
    plain_fast = fused.conv_flavor(max_c, g, n_out=n_out)             # fastest plain: imma2x2
    plain_core = fused.conv_flavor(max_c, g, allow_imma=False)        # i32
    taps = {f: D.taps_tensor(g, f) for f in {flavor, core_flavor, plain_same, plain_fast, plain_core}}
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
                     y_begin=y_begin, n_out=n_out, out=d_dev, mismatch=mismatch, imma_table=tables[fl])

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
    plain(plain_same)
    plain_kernels = {"plain_same_kernel": D.last_conv_kernel()}
    plain(plain_fast)
    plain_kernels["plain_fastest"] = D.last_conv_kernel()
    fused_step()
    kernel_kind = D.last_conv_kernel()
    torch.cuda.synchronize(dev)

    exact = None
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

    # ---------------- overhead: the plain convolutions timed like `value` ----------------
    # K back-to-back launches each on the same stream, CUDA events around them
    # (the protocol of the timed region), the blocks alternated B2B_ROUNDS
    # times and each candidate's median taken, so every leg sees the same box state
    rounds = {"entangled": [], "plain_same_kernel": [], "plain_fastest": []}
    blocks = (("entangled", fused_step), ("plain_same_kernel", lambda: plain(plain_same)),
              ("plain_fastest", lambda: plain(plain_fast)))
    for _ in range(B2B_ROUNDS):
        for name, fn in blocks:
            rounds[name].append(timed_ms(fn, stream, args.steps))
    b2b = {k: float(np.median(v)) for k, v in rounds.items()}
    cands = {
        "entangled": lambda: fused_step(flavor),
        "entangled_failed_r1": lambda: failed_step(1),
        "plain_same_kernel": lambda: plain(plain_same),
        "plain_fastest": lambda: plain(plain_fast),
        "entangled_cuda_core": lambda: fused_step(core_flavor),
        "plain_cuda_core_same_width": lambda: plain(core_flavor),
    }
    # every launch timed on its own, the candidates' order rotated from round to round: what a
    # launch costs depends on its predecessor (behind the 1 ms F64 kernels, whose int64 output
    # is still being written back from L2, the m = 3 kernel's first tiles take 5 us longer), so
    # each candidate gets each position equally often
    evs = {k: [] for k in cands}
    names = list(cands)
    for rnd in range(len(names) * (2 if args.steps >= 12 else 1)):
        for j in range(len(names)):
            k = names[(j + rnd) % len(names)]
            evs[k].append(event_time(cands[k], stream))
    torch.cuda.synchronize(dev)
    t = {k: [a.elapsed_time(b) for a, b in v] for k, v in evs.items()}
    med = {k: statistics.median(v) for k, v in t.items()}

    def ovh(a, b):
        return statistics.median([(x - y) / y * 100 for x, y in zip(t[a], t[b])])

    overhead_pct = (b2b["entangled"] - b2b["plain_same_kernel"]) / b2b["plain_same_kernel"] * 100
    overhead = {
        "back_to_back_ms": b2b,
        "interleaved_vs_plain_same_kernel_pct": ovh("entangled", "plain_same_kernel"),
        "vs_plain_fastest_pct": (b2b["entangled"] - b2b["plain_fastest"]) / b2b["plain_fastest"] * 100,
        "failed_r1_vs_plain_same_kernel_pct": ovh("entangled_failed_r1", "plain_same_kernel"),
        "cuda_core_same_width_pct": ovh("entangled_cuda_core", "plain_cuda_core_same_width"),
        "interleaved_ms": med,
        "flavors": {"entangled": MAC_NAMES[flavor], "plain_same_kernel": MAC_NAMES[plain_same],
                    "plain_fastest": MAC_NAMES[plain_fast], "cuda_core": MAC_NAMES[core_flavor]},
        "kernels": dict(plain_kernels, entangled=kernel_kind),
        "plain_fastest_samples_per_s": samples_job / (b2b["plain_fastest"] / 1e3) if world == 1 else None,
    }

    # ---------------- measured pipe peaks (roofline denominators) ----------------
    peaks = {}
    for kind in (BENCH_TC05, BENCH_IMMA, MAC_F64):
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
    # fused launch per step, back to back on `stream`)
    kern_ms = ms_step
    macs_alg = m * n * K                      # M*N*K
    digit_macs = macs_alg * np_ * ng          # int8 digit products the method needs
    achieved = 2 * digit_macs / (kern_ms / 1e3) / 1e12
    tc = kernel_kind.startswith("tcgen05")
    peak = 2 * peaks["tcgen05_i8" if tc else "imma_s8_mma_sync"] / 1e12
    kt = (K + 127 + 127) // 128 * 128      # tcgen05 Toeplitz band: K + 127 padded to 128
    issued_macs = m * (n + K - 1) * kt * np_ * ng if tc else None
    hbm, hbm_src = hbm_peak()
    io_bytes = m * (n_in + n_out) * 4  # int32 streams in, int32 recovered outputs out
    traffic = None
    tf = REPO / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(kernel_kind, {}).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "kernel": kernel_kind, "flavor": MAC_NAMES[flavor],
                "algorithmic_per_launch": {"conv_macs": macs_alg, "digit_planes": np_, "tap_digits": ng,
                                           "digit_macs": digit_macs, "tensor_macs_issued": issued_macs,
                                           "hbm_bytes": io_bytes},
                "issued_frac": (2 * issued_macs / (kern_ms / 1e3) / 1e12 / peak) if issued_macs else None,
                "hbm_gb_s": io_bytes / (kern_ms / 1e3) / 1e9, "hbm_frac": io_bytes / (kern_ms / 1e3) / 1e9 / hbm,
                "hbm_peak_gb_s": hbm, "hbm_peak_source": hbm_src,
                "peak_source": "measured in this run: nent_microbench tcgen05.mma kind::i8 128x128x32 chains, "
                               "1 CTA/SM" if tc else "measured in this run: mma.sync s8 microbench",
                "peaks_measured_gmac_s": {k: v / 1e9 for k, v in peaks.items()}}

    # ---------------- e2e through the host-buffer path ----------------
    e2e = run_e2e(params, g, flavor, x_dev, d_dev, c_np, world, rank, y_begin, n_out, samples_job, dev, xdev)
    api = run_api_e2e(params, c_np, g, dev) if (rank == 0 and world == 1 and not args.no_extras) else None

    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = other_configs(D, fused, dev, stream, args.w)
        extras["codec_passes"] = codec_passes(D, dev, stream, params, c_dev, g)
        extras["geometry_ab"] = geometry_ab(D, dev, stream, c_dev, g, args.w)
    spg = None
    if world in (4, 8) and not args.no_extras:
        del d_dev, y_plain
        torch.cuda.empty_cache()
        try:  # an extra: a failure here must not cost the halo-split headline line
            spg = run_stream_per_gpu(3 if world == 4 else 5, min(args.steps, 20), args.warmup, dev, backend)
        except Exception as exc:  # pragma: no cover - multi-GPU only
            spg = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c_np, g, params, args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "overhead_pct": overhead_pct,
            "exact": exact, "mismatches": int(mismatch.item()),
            "dtype": "int8 digits x int8 digits -> int32 -> int64 (exact integer; int32 in/out)",
            "data": "synthetic (canonical seeded cfg2 draw, SURVEY.md 8d)",
            "config": bench_config(world, args.w),
            "overhead": overhead,
            "roofline": roofline,
            "e2e": e2e,
            "e2e_numpy_api": api,
            "gpu_launches": args.steps,  # one fused kernel per step (tap table prepared before)
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "stream_per_gpu": spg,
            "other_configs": extras,
        }
        # the figures a reader of the line's tail needs, repeated as its last key
        out["summary"] = {
            "ms_per_step": ms_step, "value": value, "roofline_frac": roofline["frac"],
            "overhead_pct": overhead_pct,
            "overhead_interleaved_pct": overhead["interleaved_vs_plain_same_kernel_pct"],
            "overhead_vs_plain_fastest_pct": overhead["vs_plain_fastest_pct"],
            "back_to_back_ms": b2b, "e2e_value": e2e["value"], "exact": exact,
            "cfg3_ms": extras["cfg3"]["ms"] if extras else None,
            "cfg5_ms": extras["cfg5"]["ms"] if extras else None,
        }
        print(json.dumps(compact(out)))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(params, g, flavor, x_dev, d_dev, c_np, world, rank, y_begin, n_out, samples_job, dev, xdev):
    """The same metric end to end through the public host-buffer API
    (hostpath.ChunkedEntangledConv): pinned int32 host input -> H2D -> fused
    kernel -> D2H of the recovered int32 outputs, every step; `reps` steps
    streamed as one CUDA graph, wall clock incl. sync, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1509_03838_b200.hostpath import ChunkedEntangledConv

    m, H = params.m, len(g) - 1
    xin_np = c_np.astype(np.int32) if world == 1 else x_dev.cpu().numpy()  # [halo | slice] for N > 1
    n_e = xin_np.shape[1]
    pipe = ChunkedEntangledConv(params, n_e, g, flavor)  # 2^20-sample chunks, output lag 1
    c_host = torch.from_numpy(xin_np).pin_memory()
    d_host = torch.empty((m, n_e + H), dtype=torch.int32).pin_memory()
    o0 = 0 if world == 1 else y_begin  # this rank's outputs inside the pipeline's full conv

    def shard_ok() -> bool:
        return bool(torch.equal(d_host[:, o0:o0 + n_out], d_dev.cpu()))

    reps = 8
    pipe.capture(c_host, d_host)
    d_host.zero_()
    pipe.replay()
    torch.cuda.synchronize(dev)
    ok = shard_ok()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(3):
        pipe.replay()
        torch.cuda.synchronize(dev)
    single_s = (time.perf_counter() - t0) / 3
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
    return {"value": samples_job / e2e_s, "unit": UNIT, "h2d_bytes_per_step": pipe.h2d_bytes() * world,
            "d2h_bytes_per_step": pipe.d2h_bytes() * world, "ms_per_step": e2e_s * 1e3,
            "steps_streamed": reps, "single_step_ms": single_s * 1e3, "bit_exact_vs_device_output": bad == 0.0,
            "path": "hostpath.ChunkedEntangledConv: pinned int32 host -> chunked H2D / fused kernel / D2H "
                    "on 3 streams, steps captured as one CUDA graph (DESIGN.md 7)",
            "kernels_per_step": pipe.launches // reps}


def run_api_e2e(params, c_np, g, dev):
    """The drop-in call a reference user makes, timed end to end:
    fused.entangled_conv(StreamBlock(params, int64 numpy)) -> int64 numpy
    (pageable copies both ways, flavour chosen from the data's bound)."""
    import torch

    import paper_1509_03838_b200 as nent
    from paper_1509_03838_b200 import fused

    block = nent.StreamBlock(params, c_np)
    res = fused.entangled_conv(block, g)  # warm-up
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = fused.entangled_conv(block, g)
        ts.append(time.perf_counter() - t0)
    known = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())["cfg2"]["d"]
    s = min(ts)
    samples = res.outputs.data.size
    return {"value": samples / s, "unit": UNIT, "ms_per_call": s * 1e3,
            "h2d_bytes_per_step": int(c_np.nbytes), "d2h_bytes_per_step": int(res.outputs.data.nbytes),
            "exact": sha(res.outputs.data) == known and res.mismatches == 0,
            "call": "fused.entangled_conv(StreamBlock(params, numpy int64 (3, 2^24)), g) -> numpy int64",
            "flavor": res.flavor}


def codec_passes(D, dev, stream, params, c_dev, g):
    """K1 (entangle) and K3 (extract) alone on cfg2-sized streams, against the
    HBM roofline: bytes moved per launch / launch time."""
    import torch

    hbm, _ = hbm_peak()
    m, n = c_dev.shape
    res = {}
    eps = torch.empty((m, n), dtype=torch.int32, device=dev)
    ms = timed_ms(lambda: D.entangle(c_dev, params.l, out_dtype=torch.int32, out=eps), stream, 20)
    byts = m * n * 4 * 2  # read c (each sample once from HBM; c_{i-1} hits L2), write eps
    res["entangle_k1"] = {"ms": ms, "gb_s": byts / (ms / 1e3) / 1e9, "hbm_frac": byts / (ms / 1e3) / 1e9 / hbm,
                          "bytes": byts, "shape": "3 x 2^24 int32 -> int32"}
    delta = torch.empty((m, n), dtype=torch.int64, device=dev)
    delta.copy_(eps)  # any consistent words do: the pass's cost does not depend on the values
    out = torch.empty((m, n), dtype=torch.int32, device=dev)
    for r in (0, 1):
        ms = timed_ms(lambda: D.extract(delta, m, params.l, r, wide=params.w > 32, out=out,
                                        check_overflow=False), stream, 20)
        byts = (m - 1) * n * 8 + m * n * 4
        res[f"extract_k3_r{r}"] = {"ms": ms, "gb_s": byts / (ms / 1e3) / 1e9,
                                   "hbm_frac": byts / (ms / 1e3) / 1e9 / hbm, "bytes": byts,
                                   "shape": "2 surviving int64 rows of 2^24 -> 3 int32 rows"}
    return res


def geometry_ab(D, dev, stream, c_dev, g, w):
    """The cfg2 fused kernel at the other codec geometry (same recovered
    outputs; 5 digit planes at w=64 vs 4 at w=48)."""
    import torch

    import paper_1509_03838_b200 as nent
    from paper_1509_03838_b200._lib import MAC_NAMES, imma_flavor

    other = 64 if w == 48 else 48
    p = nent.derive_params(3, other)
    m, n = c_dev.shape
    K = len(g)
    fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(int(np.abs(g).max())))
    gd = D.taps_tensor(g, fl)
    tab = D.imma_table(gd, K, fl, 0)
    L = n + K - 1
    out = torch.empty((m, (L + 31) // 32 * 32), dtype=torch.int32, device=dev)[:, :L]
    mm = torch.zeros(1, dtype=torch.int64, device=dev)
    f = lambda: D.fused_conv(c_dev, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm,  # noqa: E731
                             imma_table=tab)
    ms = timed_ms(f, stream, 20)
    kern = D.last_conv_kernel()
    known = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())["cfg2"]["d"]
    ok = sha(out.to(torch.int64).cpu().numpy()) == known and int(mm.item()) == 0
    return {"geometry": f"({p.m},{p.w},{p.l},{p.k})", "flavor": MAC_NAMES[fl], "kernel": kern, "ms": ms,
            "samples_per_s": m * L / (ms / 1e3), "exact": ok}


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



def other_configs(D, fused, dev, stream, w):
    """The other BASELINE configs through the same fused path on one GPU:
    ms per launch, output samples/s, and the known-answer digest check (no
    failure); cfg4 inner and outer products against the HBM roofline."""
    import torch

    from paper_1509_03838_b200 import workloads
    from paper_1509_03838_b200._lib import MAC_G64, MAC_NAMES

    hbm, hbm_src = hbm_peak()
    digests = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())
    res = {}
    for cfg in (1, 3, 5):
        wl = workloads.make(cfg)
        p = wl.params
        c = torch.from_numpy(wl.c).to(dev).to(torch.int32)
        n, K = wl.n, wl.K
        L = n + K - 1
        out = D.alloc_rows(wl.m, L, torch.int32, dev)  # 128-byte aligned rows, what the device API allocates
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
        # (the fused m = 8 tcgen05 kernel takes cfg5's chain rows; NENT_BENCH_CFG5_SPLIT=1
        # times the older plain conv + separate extract pass instead)
        split = (chain and D.imma_kernel(fl, K, wl.m, False) == "tcgen05"
                 and (D.imma_kernel(fl, K, wl.m, True) != "tcgen05"
                      or os.environ.get("NENT_BENCH_CFG5_SPLIT") == "1"))
        if split:
            delta = D.alloc_rows(wl.m, L, torch.int32, dev)

        def run():
            if chain:
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
        kern = D.last_conv_kernel()
        ok = sha(out.to(torch.int64).cpu().numpy()) == digests[f"cfg{cfg}"]["d"] and int(mm.item()) == 0
        ms = timed_ms(run, stream, 20 if chain else 50)  # back-to-back launches, the headline's protocol
        res[f"cfg{cfg}"] = {"flavor": MAC_NAMES[fl], "ms": ms, "kernel": ("tcgen05 conv + verifying extract"
                                                                          if split else kern),
                            "samples_per_s": wl.m * L / (ms / 1e3), "conv_gmac_s": wl.m * n * K / (ms / 1e3) / 1e9,
                            "exact": ok}
        if chain:  # per-pass breakdown of the chain (bytes moved / time)
            passes = {"interleave_chain": (lambda: D.interleave_chain(c, p.l, wl.scale, add, out=ct),
                                           2 * wl.m * n * 4 + n * 8),
                      "gather_records": (lambda: D.gather_records(ct, perm, out=xg), 2 * wl.m * n * 4 + n * 4)}
            if split:
                passes["conv"] = (lambda: D.conv(xg, gd, K, fl, period=L, n_out=L, out=delta), 2 * wl.m * n * 4)
                passes["extract_verify"] = (lambda: D.extract_verify(delta, wl.m, p.l, 0, p.w > 32, mm, out=out),
                                            2 * wl.m * L * 4)
            else:
                passes["fused_conv_extract"] = (lambda: D.fused_conv(xg, gd, K, p.l, fl, None, True, L, n_in=n,
                                                                     out=out, mismatch=mm, pre_entangled=True,
                                                                     imma_table=tab), 2 * wl.m * n * 4)
            res[f"cfg{cfg}"]["passes"] = {}
            for name, (fn, byts) in passes.items():
                pms = timed_ms(fn, stream, 20)
                res[f"cfg{cfg}"]["passes"][name] = {"ms": pms, "bytes": byts, "gb_s": byts / (pms / 1e3) / 1e9,
                                                    "hbm_frac": byts / (pms / 1e3) / 1e9 / hbm}
        del c, out
        torch.cuda.empty_cache()
    # cfg4 inner products (65,536 x 4,096 per stream, 3 streams)
    wl = workloads.make(4)
    c = torch.from_numpy(wl.c).to(dev).to(torch.int32)
    r = fused.entangled_inner(wl.params, c, wl.g)  # public API once: digest + redundant check
    ok = sha(r.outputs.data.to(torch.int64).cpu().numpy()) == digests["cfg4_inner"]["d"] and r.mismatches == 0
    gd = D.taps_tensor(wl.g, MAC_G64)

    def inner():
        D.fused_inner(c, gd, wl.params.l, None, True, MAC_G64, out_dtype=torch.int64)

    ms = timed_ms(inner, stream, 5)
    res["cfg4_inner"] = {"flavor": r.flavor, "ms": ms, "hbm_gb_s": c.numel() * 4 / (ms / 1e3) / 1e9,
                         "hbm_frac": c.numel() * 4 / (ms / 1e3) / 1e9 / hbm, "hbm_peak_source": hbm_src,
                         "exact": ok}
    # cfg4 outer products: d[i, b, u, v] = c[i, b, u] g[v] recovered through the
    # entangled domain; 3.3e12 outputs for the whole batch (26 TB as int64), so
    # a window of B vectors is materialised (int32) into one reused buffer and
    # timed against the HBM store roofline; the full batch is extrapolated
    B = 16
    n4 = wl.c.shape[2]
    outo = torch.empty((3, B, n4, n4), dtype=torch.int32, device=dev)
    cw = c[:, :B].contiguous()
    ms = timed_ms(lambda: fused.entangled_outer(wl.params, cw, wl.g, out=outo), stream, 3)
    ref = wl.c[:, :2, :, None] * wl.g[None, None, None, :]  # vectors 0 and 1 elementwise
    ok = bool(np.array_equal(outo[:, :2].to(torch.int64).cpu().numpy(), ref))
    store = outo.numel() * 4
    res["cfg4_outer"] = {"vectors_timed": B, "ms": ms, "outputs_per_s": outo.numel() / (ms / 1e3),
                         "store_gb_s": store / (ms / 1e3) / 1e9, "hbm_frac": store / (ms / 1e3) / 1e9 / hbm,
                         "full_batch_s_extrapolated": ms / 1e3 * wl.c.shape[1] / B,
                         "exact_vectors_0_1": ok, "out_dtype": "int32"}
    del c, cw, outo
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



def reference_package_sample(c, g, params, seconds: float = 8.0):
    """The reference package itself (baseline/_ref: the unmodified `nent`,
    numpy + numba, single-threaded by design) on a bounded cfg2 sample through
    its public API: entangle -> apply_entangled(CIRCULAR_CONVOLUTION on the
    zero-padded streams) -> disentangle(failed=None), the stages its own
    bench.py times (pkg/src/nent/bench.py:74-125).  None when not installed."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "nent").is_dir():
        return None
    code = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import nent
c = np.load(sys.argv[2]); g = np.load(sys.argv[3])
p = nent.CodecParams(*[int(v) for v in sys.argv[4].split(",")])
budget = float(sys.argv[5])
K = len(g)
def run(ns):
    pad = np.zeros((c.shape[0], ns + K - 1), dtype=np.int64); pad[:, :ns] = c[:, :ns]
    op = nent.LsbOp(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector(g))
    t0 = time.perf_counter()
    e = nent.entangle(nent.StreamBlock(p, pad))
    d = nent.apply_entangled(op, e)
    out = nent.disentangle(d, failed=None)
    t = time.perf_counter() - t0
    t1 = time.perf_counter(); plain = nent.apply_conventional(op, nent.StreamBlock(p, pad)); tp = time.perf_counter() - t1
    assert np.array_equal(out.data, plain.data)
    return t, tp, out.data.size
ns = 1 << 12
t, tp, s = run(ns)
ns = int(min(c.shape[1], max(ns, ns * budget / max(t, 1e-6))))
t, tp, s = run(ns)
print(json.dumps({"value": s / t, "plain_value": s / tp, "seconds": t + tp, "samples_per_stream": ns}))
"""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        cp, gp = Path(td) / "c.npy", Path(td) / "g.npy"
        np.save(cp, np.ascontiguousarray(c[:, : 1 << 20]))
        np.save(gp, g)
        try:
            r = subprocess.run([sys.executable, "-c", code, str(ref), str(cp), str(gp),
                                f"{params.m},{params.w},{params.l},{params.k}", str(seconds)],
                               capture_output=True, text=True, timeout=600,
                               env=dict(os.environ, OMP_NUM_THREADS="1", NUMBA_NUM_THREADS="1"))
            out = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:  # pragma: no cover - reported, not fatal
            return {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    return {"value": out["value"], "unit": UNIT, "cores": 1, "kind": "reference",
            "plain_value": out["plain_value"], "overhead_pct": (out["plain_value"] / out["value"] - 1) * 100,
            "sample": f"first {out['samples_per_stream']} samples of each cfg2 stream through the unmodified "
                      "nent package (baseline/_ref, numpy + numba, 1 thread): entangle -> apply_entangled(conv "
                      "of the zero-padded streams) -> disentangle(failed=None)",
            "seconds": out["seconds"]}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # only rank 0 runs the CPU reference arm
    from oracle import oracle as O

    params, c, g = make_inputs(0, 1 << 24, 256, args.w)
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
    pkg = reference_package_sample(c, g, params)
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64 (reference numpy semantics)",
        "data": "synthetic (canonical seeded cfg2 draw, SURVEY.md 8d)",
        "config": bench_config(world, args.w),
        "impl": "reference",
        "overhead_pct": statistics.median([(a - b) / b * 100 for a, b in zip(te, tp)]),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"first {ns} samples of each cfg2 stream per step (K=256, full "
                                   f"conv, entangle+conv+recover), oracle/nent_oracle.c OpenMP",
                         "host": host_desc(), "reference_package": pkg},
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
