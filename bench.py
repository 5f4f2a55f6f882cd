#!/usr/bin/env python
"""bench.py -- batched DeepInverse recovery throughput on B200 (BASELINE.json `metric`).

One *step* = one di_recover of a whole per-GPU batch: y -> x_tilde = Phi^T y -> conv 1->64+ReLU ->
conv 64->32+ReLU -> conv 32->1 -> x_hat (every row of SURVEY.md §8(a)), inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config lowrate] [--impl ours|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...   (one rank per GPU)

Multi-GPU: the images are independent, so rank r recovers global images
[r*B, (r+1)*B) with Phi and Omega replicated and NO collective on the data path ("scaling": "weak").
torch.distributed (NCCL) only aligns the start (barrier) and takes the max of the per-rank device times.

Rank 0 prints ONE JSON line.  `value` = images recovered by all ranks / max-over-ranks device time;
`e2e` = the same through di_recover_host (pinned host y in, host x_hat out, copies inside the timed
region); `roofline` = the dominant kernel (conv layer 2) measured live with CUDA events recorded by the
library on the launching stream; `cpu_baseline` = the fp64 oracle (oracle/, test infrastructure) timed
as it stands on this host's cores over a bounded sample of the same workload.

`--impl reference`: this tier has no reference implementation; the reference arm is the oracle, run on
the host cores over a bounded sample per step (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "recovered images/sec per GPU and 8-GPU; achieved tensor-core TFLOP/s vs peak"
UNIT = "images/s"
KSZ = 11
CONV2_FLOP_PER_PX = 2 * 32 * 64 * KSZ * KSZ          # 495 616
PATH_FLOP_PER_PX = 2 * (64 * 1 + 32 * 64 + 1 * 32) * KSZ * KSZ   # 2 * 259 424 conv taps


# ----------------------------------------------------------------------------- distributed plumbing
def dist_env() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process when absent)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(rank: int, per_rank: int) -> tuple[int, int]:
    """Global image indices [start, stop) recovered by `rank` (contiguous blocks, weak scaling)."""
    return rank * per_rank, (rank + 1) * per_rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def aggregate(per_rank_units: int, world: int, max_seconds: float) -> float:
    """Whole-job throughput: units of all ranks / slowest rank's time."""
    return per_rank_units * world / max_seconds


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launcher_cmd(argv: list[str], gpus: int, port: int) -> list[str]:
    """The command `python bench.py --gpus N` re-executes itself under: torchrun, one rank per GPU, loopback
    rendezvous (the container hostname may not resolve)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def gather_to_all(t, world: int) -> list:
    """all_gather of one same-shape tensor per rank (NCCL on the GPU box, gloo in the CPU tests) -- checking only,
    outside the timed region."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return [t]
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return parts


def check_rows(batch: int, k: int = 32) -> list[int]:
    """Local image indices a rank's outputs are checked on: the first and last k (all when batch <= 2k)."""
    if batch <= 2 * k:
        return list(range(batch))
    return list(range(k)) + list(range(batch - k, batch))


# ----------------------------------------------------------------------------- clocks (nvidia-smi)
_CLK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
_REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
# the remaining nvmlClocksEventReason bits (nvml.h), reported as `other_clock_events`
_OTHER_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x10: "sync_boost",
                  0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


_NVML_LOOP = r"""
import sys, time
import pynvml as nv
gpu, path = int(sys.argv[1]), sys.argv[2]
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(gpu)
bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
with open(path, "w", buffering=1) as f:
    while True:
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        try:     # instantaneous draw: nvmlDeviceGetPowerUsage is an average that lags a 0.14-s timed region
            pi = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
            pin = pi.value.uiVal / 1000.0 if pi.nvmlReturn == 0 else -1.0
        except Exception:
            pin = -1.0
        f.write("%.6f,%d,%d,%.3f,%s,%.3f,%d\n" % (time.time(), sm, mx, pw,
                                                  ",".join("1" if rs & b else "0" for b in bits), pin, rs))
        time.sleep(0.004)
"""


class ClockSampler:
    """Samples SM clock, power and throttle reasons every ~5 ms while the timed region runs -- the
    B200_PROFILING.md clocks line.  The NVML loop runs in its own PROCESS (a thread would compete with the timing
    loop for the GIL and can miss the whole region); rows are timestamped and only those inside the region are
    kept.  Fallback: nvidia-smi -lms 200."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.kind = None
        self.t0 = self.t1 = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            import pynvml  # noqa: F401  (the child imports it; fail here to use the fallback)
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_LOOP, str(self.gpu), self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            self.kind = "nvml"
        except Exception:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={_CLK_FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            self.kind = "nvidia-smi"
        deadline = time.time() + 20.0      # wait for the first sample (the child's imports)
        while time.time() < deadline and os.path.getsize(self.path) == 0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        time.sleep(0.02)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.kind == "nvidia-smi":
            self.fh.close()

    def summary(self) -> dict:
        rows, inside = [], []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                try:
                    if self.kind == "nvml" and len(f) >= 8:
                        pin = float(f[8]) if len(f) >= 10 else -1.0
                        mask = int(f[9]) if len(f) >= 10 else 0
                        # r[2]: the draw that decides "under load" -- instantaneous when NVML reports it
                        r = (float(f[1]), float(f[2]), pin if pin >= 0 else float(f[3]), [v == "1" for v in f[4:8]],
                             float(f[3]), mask)
                        rows.append(r)
                        if self.t0 <= float(f[0]) <= self.t1:
                            inside.append(r)
                    elif self.kind == "nvidia-smi" and len(f) >= 9:
                        pw = float(f[3]) if f[3] not in ("", "[N/A]") else 0.0
                        rows.append((float(f[1]), float(f[2]), pw, [v.lower().startswith("active") for v in f[5:9]],
                                     pw, 0))
                except ValueError:
                    continue
            os.unlink(self.path)
        rows = inside or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        # rows inside the timed region are under load by construction (the steps are queued back to back between two
        # synchronisations); NVML's power readings -- averaged AND "instantaneous" -- lag a 0.14-s region by up to
        # ~0.1 s, so filtering on them kept only the late, already power-capped samples.  Without timestamps (the
        # nvidia-smi fallback, or no row inside) fall back to the draw.
        load = rows if inside else ([r for r in rows if r[2] > 300.0] or rows)
        reasons = sorted({_REASONS[i] for r in load for i, v in enumerate(r[3]) if v})
        # every other NVML clocks-event bit seen under load, by name, so that a clock below max never reads as
        # "no reason" only because the reason is not one of the four above
        mask = 0
        for r in load:
            mask |= r[5]
        other = sorted(n for b, n in _OTHER_REASONS.items() if mask & b)
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "other_clock_events": other, "samples": len(rows),
                "samples_under_load": len(load), "power_w_max": max(r[2] for r in rows),
                "power_avg_w_max": max(r[4] for r in rows), "sampler": self.kind,
                "window": "timed region only" if inside else "whole sampler run"}


def _conv2_tiles(L: int):
    """Output counts of k_conv2_tc's tiles for a unit of L strip positions: ceil(L / 253) tiles sharing the outputs
    evenly, or -- when that saves MMA columns -- first tiles one 16-column step shorter and the rest in the last."""
    r16 = lambda x: (x + 15) // 16 * 16
    nt = -(-L // 253)
    s = -(-L // nt)
    sf = (s + 3) // 16 * 16 - 3
    lf = L - (nt - 1) * sf
    cols = lambda sp, last: (nt - 1) * r16(sp + 3) + r16(last + 3)
    if sf > 0 and lf <= 253 and cols(sf, lf) < cols(s, L - (nt - 1) * s):
        s = sf
    return [s] * (nt - 1) + [L - (nt - 1) * s]


def conv2_row_blocks(n1: int, n2: int, rows: int = 6):
    """k_conv2_tc's row blocks (r0, height): `rows`-row blocks and a short last one, or (one column segment) ntall
    blocks of rows + 1 then rows-row ones when every block runs the same number of tiles and the image needs fewer
    tiles (mixed row-block heights)."""
    wseg = min(n2, 64)
    P = n2 + 5 if n2 <= 64 else wseg + 10
    uni = [(r0, min(rows, n1 - r0)) for r0 in range(0, n1, rows)]
    nrb = (n1 + rows) // (rows + 1)
    ntall = n1 - rows * nrb
    ntl = lambda h: len(_conv2_tiles((h - 1) * P + wseg))
    if n2 > 64 or not 0 < ntall <= nrb or ntl(rows + 1) != ntl(rows):
        return uni
    mixed, r0 = [], 0
    for rb in range(nrb):
        h = rows + (rb < ntall)
        mixed.append((r0, h))
        r0 += h
    return mixed if sum(ntl(h) for _, h in mixed) < sum(ntl(h) for _, h in uni) else uni


def conv2_useful_mac_ceiling(n1: int, n2: int, rows: int = 6) -> float:
    """Fraction of the tensor-core MACs k_conv2_tc issues that are useful: 11 of 12 column-tap slots,
    times output positions over MMA columns -- row blocks of conv2_row_blocks x <= 64 columns, strip pitch n2 + 5 (one
    column segment) or 74, tiles of _conv2_tiles, each issued as N = round16(count + 3) <= 256 columns."""
    wseg = min(n2, 64)
    ncs = -(-n2 // wseg)
    P = n2 + 5 if ncs == 1 else wseg + 10
    useful = cols = 0
    for _, rr in conv2_row_blocks(n1, n2, rows):
        L = (rr - 1) * P + wseg
        for cnt in _conv2_tiles(L):
            cols += min(256, (cnt + 3 + 15) // 16 * 16)
        useful += rr * wseg
    return 11.0 / 12.0 * useful / cols


# ----------------------------------------------------------------------------- workload
def workload(name: str):
    import synth
    c = synth.CONFIGS[name]
    prec = c.precisions[-1] if name != "paper" else "tf32"
    return c, prec


def make_inputs(c, prec: str, start: int, count: int):
    """Seeded synthetic inputs of the config; global image indices start..start+count-1."""
    import synth
    st = "bf16" if prec == "bf16" else "f32"
    phi = synth.make_phi(c.m, c.N, st)
    x = synth.make_images(c.n, start, count, c.n_blobs, c.n_rects, c.texture_var)
    y = synth.measure(phi, x, st)
    params = synth.make_params().rounded(st)
    return phi, x, y, params


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16_tflops": d["bf16_tflops"], "bf16_tflops_sustained": d.get("bf16_tflops_sustained"),
                "hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


def traffic_for(kernel: str, config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(f"{kernel}@{config}")
    return e.get("bytes_per_launch") if e else None


# ----------------------------------------------------------------------------- CPU oracle timing
def oracle_sample(c, prec: str, budget_s: float, threads: int, max_images: int | None = None) -> dict:
    """Time the fp64 oracle (as it stands) on the first images of the workload, in chunks of `threads`
    images (OpenMP over images), until `budget_s` of wall time is used.  Returns images/s."""
    import oracle
    phi, x, y, params = make_inputs(c, prec, 0, threads)
    done, t_total = 0, 0.0
    while True:
        t0 = time.perf_counter()
        oracle.forward(y, phi, params, c.n, c.n, threads=threads)
        t_total += time.perf_counter() - t0
        done += y.shape[0]
        if t_total >= budget_s or (max_images is not None and done >= max_images):
            break
    # single thread, per image: 2 images on one core
    t0 = time.perf_counter()
    oracle.forward(y[:2], phi, params, c.n, c.n, threads=1)
    s1 = (time.perf_counter() - t0) / 2
    return {"value": done / t_total, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{done} images of workload {c.name} ({c.n}x{c.n}, M={c.m}) in chunks of {threads} "
                      f"(one per OpenMP thread), fp64, {t_total:.1f} s",
            "single_thread_s_per_image": s1}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    c, prec = workload(args.config)
    threads = os.cpu_count() or 1
    import oracle
    phi, x, y, params = make_inputs(c, prec, 0, threads)
    for _ in range(args.warmup):
        oracle.forward(y[:1], phi, params, c.n, c.n, threads=1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.forward(y, phi, params, c.n, c.n, threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps * y.shape[0] / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(c, prec, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{y.shape[0]} images of {c.name} per step (one per OpenMP thread), "
                                       f"fp64 C oracle, {args.steps} steps"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(c, prec, world):
    return {"workload": f"{c.name}: {c.n}x{c.n} images (N={c.N}), M={c.m} (M/N={c.m / c.N:.3g}), "
                        f"batch {c.batch}/GPU, {prec}",
            "n": c.n, "m": c.m, "batch_per_gpu": c.batch, "global_batch": c.batch * world,
            "precision": prec, "layers": "Phi^T | 64@11x11x1+ReLU | 32@11x11x64+ReLU | 1@11x11x32",
            "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
            "l2": "inputs larger than L2: per-step working set h1+h2 = "
                  f"{c.batch * c.N * 96 * (2 if prec == 'bf16' else 4) / 1e9:.2f} GB >> 126 MB L2"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1701_03891_b200 import DeepInverse, build as _b  # noqa: F401
    import paper_1701_03891_b200.build as pb
    pb.build()

    c, prec = workload(args.config)
    B = args.batch or c.batch
    lo, hi = shard(rank, B)
    phi, x, y, params = make_inputs(c, prec, lo, B)
    ctx = DeepInverse(phi, params, c.n, c.n, prec, device=local, max_batch=B)
    sdt = ctx.storage_dtype
    y_dev = torch.from_numpy(y).to(device=dev, dtype=sdt)
    xhat = torch.empty((B, c.n, c.n), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 0)):
        ctx.recover(y_dev, xhat)
    torch.cuda.synchronize(dev)

    # ---------------- device-resident timed region
    ctx.set_profiling(True)
    ctx.stage_times(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(dev)
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.recover(y_dev, xhat)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(dev)
    ms = ev0.elapsed_time(ev1)
    stage_ms, calls = ctx.stage_times(reset=True)
    ctx.set_profiling(False)
    clocks = clk.summary()
    launches = ctx.info()["launches_per_recover"] * args.steps
    t_max = max_over_ranks(ms / 1e3, dev)
    value = aggregate(B * args.steps, world, t_max)

    # ---------------- end to end through the public host API (pinned y in, host x_hat out)
    y_host = torch.from_numpy(y).to(dtype=sdt).pin_memory()
    x_host = torch.empty((B, c.n, c.n), dtype=torch.float32).pin_memory()
    for _ in range(max(args.warmup, 1)):
        ctx.recover_host(y_host, x_host.numpy())
    barrier(dev)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ctx.recover_host(y_host, x_host.numpy())
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_t = max_over_ranks(e0.elapsed_time(e1) / 1e3, dev)
    e2e = {"value": aggregate(B * args.steps, world, e2e_t), "unit": UNIT,
           "h2d_bytes_per_step": int(y_host.numel() * y_host.element_size()),
           "d2h_bytes_per_step": int(x_host.numel() * x_host.element_size())}

    # ---------------- dominant kernel roofline (conv layer 2), live CUDA events on the launching stream
    pk = peaks()
    conv2_ms = stage_ms[2] / max(calls, 1)
    conv2_flop = CONV2_FLOP_PER_PX * B * c.N
    achieved = conv2_flop / (conv2_ms / 1e3) / 1e12
    if prec == "bf16":
        peak = pk["bf16_tflops"]
        peak_note = f"bf16 dense, burst, {pk['source']}"
    elif prec == "tf32":
        peak = pk["bf16_tflops"] / 2
        peak_note = f"tf32 = measured bf16 burst x 1/2 (nominal 1.1 / 2.25 PF), {pk['source']}"
    else:
        peak = None
        peak_note = "fp32 SIMT path"
    kname = ctx.info()["stage_kernels"][2]
    roof = {"kernel": kname, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if peak else None,
            "frac_of_sustained": (achieved / pk["bf16_tflops_sustained"])
            if (peak and prec == "bf16" and pk.get("bf16_tflops_sustained")) else None,
            "peak_note": peak_note, "traffic": traffic_for(kname, c.name),
            "algorithmic": f"2*32*64*121 = {CONV2_FLOP_PER_PX} FLOP/pixel x {B * c.N} pixels per launch",
            "launch_ms": conv2_ms}
    if prec == "bf16":   # the tap-stacked form's useful-MAC ceiling and the fraction of it reached
        ceil = conv2_useful_mac_ceiling(c.n, c.n)
        roof["design_ceiling"] = ceil
        roof["frac_of_design_ceiling"] = roof["frac"] / ceil if roof["frac"] else None
        # like-for-like with the clock the kernel ran at: the dense bf16 rate of 148 SMs x 8192 FLOP/clk at the SM
        # clock sampled during the timed region (MEASURED_PEAKS' burst figure was taken at a lower, power-capped
        # clock, so `frac` alone flatters the kernel)
        if clocks.get("sm_mhz"):
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            clk_peak = nsm * 8192 * clocks["sm_mhz"] * 1e6 / 1e12
            roof["peak_at_sm_clock"] = clk_peak
            roof["frac_at_sm_clock"] = achieved / clk_peak
            roof["frac_of_design_ceiling_at_sm_clock"] = achieved / clk_peak / ceil

    per_step = ms / args.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_over_ranks(per_step, dev), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": config_dict(c, prec, world), "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "clocks": clocks,
            "stages_ms": {"proxy": stage_ms[0] / max(calls, 1), "conv1": stage_ms[1] / max(calls, 1),
                          "conv2": stage_ms[2] / max(calls, 1), "conv3": stage_ms[3] / max(calls, 1)},
            "path_tflops": (PATH_FLOP_PER_PX + 2 * c.m) * c.N * B / (per_step / 1e3) / 1e12,
            "per_gpu_images_s": B / (per_step / 1e3)}
    if prec == "bf16":
        # the thin layers against HBM: algorithmic bytes = bf16 h1 written by conv1 (128 B/px) and bf16
        # h2 read + fp32 x_hat written by conv3 (64 + 4 B/px), over each kernel's mean launch time; both kernels are
        # bound by the shared-memory port, not by HBM (ncu tc + lsu shared wavefronts, profiles/r04_*)
        thin = {}
        for name, idx, bpp in (("conv1", 1, 128), ("conv3", 3, 68)):
            t = stage_ms[idx] / max(calls, 1) / 1e3
            gbs = bpp * B * c.N / t / 1e9
            thin[name] = {"achieved_GBs": gbs, "peak_GBs": pk["hbm_gbs"], "frac": gbs / pk["hbm_gbs"],
                          "bytes_per_px": bpp, "launch_ms": t * 1e3}
        line["thin_layers"] = thin

    # ---------------- sensing model and metrics around the path, device-timed
    xt_dev = torch.from_numpy(x).to(dev)
    yb = torch.empty_like(y_dev)
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ctx.measure(xt_dev, yb)
    ctx.recover_metrics(y_dev, xt_dev, xhat)
    torch.cuda.synchronize(dev)
    sev[0].record(stream)
    ctx.measure(xt_dev, yb)
    sev[1].record(stream)
    ctx.add_noise(yb, 20.0, 1701)
    sev[2].record(stream)
    mt = ctx.metrics(xhat, xt_dev)
    sev[3].record(stream)
    sev[4].record(stream)
    _, mf = ctx.recover_metrics(y_dev, xt_dev, xhat)      # recovery + metrics in one call
    sev[5].record(stream)
    torch.cuda.synchronize(dev)
    line["sensing"] = {"measure_ms": sev[0].elapsed_time(sev[1]), "noise_20db_ms": sev[1].elapsed_time(sev[2]),
                       "metrics_ms_incl_d2h": sev[2].elapsed_time(sev[3]),
                       "recover_metrics_ms_incl_d2h": sev[4].elapsed_time(sev[5]),
                       "recover_metrics_equals_separate_psnr": bool(np.allclose(mf[0], mt[0], rtol=0, atol=1e-9)),
                       "mean_psnr_db_random_init": float(np.mean(mt[0]))}

    # ---------------- sustained: the same recovery back to back for ~2 s, after the timed region -- the rate at the
    # board's power cap (the path is power-bound; the 20-step bench starts from an idle GPU)
    if not args.no_sustained:
        line["sustained"] = sustained_probe(ctx, y_dev, xhat, B, world, dev, local, stream, line["ms_per_step"] / 1e3)

    # ---------------- single-image latency (Table 1 quotes time per image): one image through the same
    # context, device-resident (CUDA events) and end to end through di_recover_host (wall clock, host buffers)
    y1 = y_dev[:1].contiguous()
    x1 = torch.empty((1, c.n, c.n), dtype=torch.float32, device=dev)
    yh1 = y_dev[:1].cpu().pin_memory()
    xh1 = torch.empty((1, c.n, c.n), dtype=torch.float32).pin_memory()
    for _ in range(5):
        ctx.recover(y1, x1)
        ctx.recover_host(yh1, xh1.numpy())
    torch.cuda.synchronize(dev)
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    for _ in range(50):
        ctx.recover(y1, x1)
    l1.record(stream)
    torch.cuda.synchronize(dev)
    tw = time.perf_counter()
    for _ in range(50):
        ctx.recover_host(yh1, xh1.numpy())
    tw = (time.perf_counter() - tw) / 50
    line["latency"] = {"batch1_device_ms": l0.elapsed_time(l1) / 50, "batch1_e2e_wall_ms": tw * 1e3,
                       "note": "one 64x64 image per call (back-to-back calls); the paper's Table 1 context figure is "
                               "0.01 s per image on its own hardware"}

    # ---------------- training step, device-timed on its own context
    if not args.no_train:
        line["training"] = train_probe(c, prec, phi, x, y, B, world, local, dev)

    # ---------------- output check (outside the timed region): gather x_hat of every rank to rank 0 (NCCL
    # all_gather -- the only use of a collective on outputs); rank 0 re-recovers the first and
    # last 32 images of every rank's block itself (bitwise: per-image results do not depend on the rank, the batch
    # or the CTA a unit lands on) and checks 2 + 2 of them per rank against the fp64 oracle
    ok = True
    if not args.no_check:
        xhat_last = xhat.clone()
        ctx.recover(y_dev, xhat)                           # the timed loop's output, once more, for the gather
        parts = gather_to_all(xhat, world)
        if rank == 0:
            line["gather_check"] = output_check(ctx, c, prec, B, world, parts, dev, args.no_oracle_check, phi, params)
            ok = line["gather_check"]["pass"] and bool(torch.equal(xhat_last, xhat))
            line["gather_check"]["repeat_bitwise"] = bool(torch.equal(xhat_last, xhat))
        del parts

    # ---------------- CPU baseline (oracle as it stands), rank 0 at N=1 only
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        line["cpu_baseline"] = oracle_sample(c, prec, args.cpu_budget, threads)
        line["cpu_baseline"]["cpu_model"] = cpu_model()
        if not args.no_cpu_configs:
            line["cpu_baseline"]["single_thread_s_per_image"] = oracle_single_thread_per_config()
    if rank == 0:
        print(json.dumps(line), flush=True)
        if not ok:
            print("output check FAILED: " + json.dumps(line["gather_check"]), file=sys.stderr)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        barrier(dev)
        dist.destroy_process_group()
    return 0 if ok else 1


def sustained_probe(ctx, y_dev, xhat, B, world, dev, local, stream, step_s, seconds=2.0) -> dict:
    """The same number of recoveries on every rank (~`seconds` at the timed region's global step time `step_s`), back
    to back with a synchronisation every 10, CUDA events over the whole run, clocks and power sampled inside it;
    whole-job images/s from the slowest rank."""
    import torch
    n = max(10, int(seconds / max(step_s, 1e-6)) // 10 * 10)
    barrier(dev)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(n // 10):
            for _ in range(10):
                ctx.recover(y_dev, xhat)
            torch.cuda.synchronize(dev)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    t = max_over_ranks(e0.elapsed_time(e1) / 1e3, dev)
    cl = clk.summary()
    return {"images_s": aggregate(B * n, world, t), "steps": n, "ms_per_step": t / n * 1e3, "seconds": t,
            "sm_mhz": cl.get("sm_mhz"), "power_w_max": cl.get("power_w_max"), "reasons": cl.get("reasons")}


def train_probe(c, prec, phi, x, y, B, world, local, dev, batch=1024, steps=10, warmup=3) -> dict:
    """One data-parallel SGD step per iteration: di_train_grad of this
    rank's first `batch` images with scale 1/global batch, the NCCL all-reduce of the gradient (the method's only
    hot collective; absent at N = 1), di_sgd_step.  Own context (the weights change), per-channel biases; CUDA events
    on the launching stream, max over ranks."""
    import torch
    import torch.distributed as dist
    import synth
    from paper_1701_03891_b200 import DeepInverse
    bt = min(batch, B)
    st = "bf16" if prec == "bf16" else "f32"
    tctx = DeepInverse(phi, synth.make_params(bias="channel").rounded(st), c.n, c.n, prec, device=local, max_batch=bt)
    yd = torch.from_numpy(y[:bt]).to(device=dev, dtype=tctx.storage_dtype)
    xd = torch.from_numpy(x[:bt]).to(dev)
    scale = 1.0 / (bt * world)
    grads = torch.empty(tctx.num_params(), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(lr):
        loss, _ = tctx.train_grad(yd, xd, scale, grads)
        if world > 1:
            dist.all_reduce(grads)
            dist.all_reduce(loss)
        tctx.sgd_step(grads, lr, 0.9)
        return loss

    loss0 = step(0.0)
    lr = 0.05 * float(loss0.item()) / max(float((grads.double() ** 2).sum()), 1e-30)
    for _ in range(warmup):
        step(lr)
    torch.cuda.synchronize(dev)
    barrier(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        loss = step(lr)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = max_over_ranks(e0.elapsed_time(e1) / 1e3, dev)
    out = {"images_s": aggregate(bt * steps, world, t), "ms_per_step": t / steps * 1e3, "batch_per_gpu": bt,
           "precision": prec, "steps": steps, "warmup": warmup, "allreduce": "nccl" if world > 1 else "none (N = 1)",
           "loss_first_last": [float(loss0.item()), float(loss.item())],
           "what": "di_train_grad (forward keeping activations, MSE loss, backprop through the 3 convs and Phi^T) "
                   "+ gradient all-reduce + di_sgd_step (momentum 0.9), per-channel biases"}
    tctx.close()
    return out


def output_check(ctx, c, prec, B, world, parts, dev, no_oracle=False, phi=None, params=None) -> dict:
    """Rank 0: bitwise equality of every rank's gathered x_hat with rank 0's own recovery of the same global images
    (first and last 32 of each block), and the oracle's rel-L2 / element-wise error on 2 + 2 of them per rank."""
    import torch
    rows = check_rows(B)
    orows = [0, 1, B - 2, B - 1] if B >= 4 else list(range(B))
    bitwise, rel_max, pix_max, n_or = True, 0.0, 0.0, 0
    tol = {"bf16": 2e-2, "tf32": 2e-2, "f32": 1e-5}[prec]
    for r in range(world):
        lo = r * B
        phi, x, y, params = make_inputs_rows(c, prec, [lo + i for i in rows], phi, params)
        yd = torch.from_numpy(y).to(device=dev, dtype=ctx.storage_dtype)
        mine = ctx.recover(yd).cpu().numpy()
        got = parts[r][rows].cpu().numpy()
        bitwise &= bool(np.array_equal(mine, got))
        if not no_oracle:
            import oracle
            sel = [rows.index(i) for i in orows]
            ref = oracle.forward(y[sel], phi, params, c.n, c.n)
            for g, rf in zip(got[sel], ref):
                rel_max = max(rel_max, oracle.rel_l2(g, rf))
                pix_max = max(pix_max, float(np.max(np.abs(g - rf)) / max(float(np.max(np.abs(rf))), 1e-30)))
                n_or += 1
    ok = bitwise and (no_oracle or (rel_max <= tol and pix_max <= tol))
    return {"ranks": world, "bitwise_images_per_rank": len(rows), "bitwise_vs_rank0_recovery": bitwise,
            "oracle_images": n_or, "oracle_max_rel_l2": rel_max, "oracle_max_pixel_err_over_max": pix_max,
            "tol": tol, "pass": ok}


def make_inputs_rows(c, prec: str, idx: list[int], phi=None, params=None):
    """Seeded inputs for an arbitrary list of global image indices (contiguous runs generated together); phi / params
    may be passed in when the caller already generated them (they depend only on the seed)."""
    import synth
    st = "bf16" if prec == "bf16" else "f32"
    if phi is None:
        phi = synth.make_phi(c.m, c.N, st)
    xs, run = [], [idx[0]]
    for i in idx[1:] + [None]:
        if i is not None and i == run[-1] + 1:
            run.append(i)
            continue
        xs.append(synth.make_images(c.n, run[0], len(run), c.n_blobs, c.n_rects, c.texture_var))
        if i is not None:
            run = [i]
    x = np.concatenate(xs)
    y = synth.measure(phi, x, st)
    return phi, x, y, (params if params is not None else synth.make_params().rounded(st))


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "?"


def oracle_single_thread_per_config() -> dict:
    """the oracle's single-thread time per image on each config (Tiny 4, Paper 16, Low-rate 16,
    Larger 4 images; Stress 1 image, extrapolated: its lifting step is timed on the first 1024 of the 16384 rows of
    Phi -- the proxy loop is linear in M -- and the convolutions on the whole image).  The five timings run
    concurrently, one host thread each (ctypes releases the GIL), so the whole takes about the longest one."""
    from concurrent.futures import ThreadPoolExecutor
    import oracle
    import synth

    def one(name, count):
        c = synth.CONFIGS[name]
        st = "bf16" if c.precisions[-1] == "bf16" else "f32"
        if name != "stress":
            phi, x, y, params = make_inputs_rows(c, "bf16" if st == "bf16" else "f32", list(range(count)))
            t0 = time.perf_counter()
            oracle.forward(y, phi, params, c.n, c.n, threads=1)
            return name, {"s_per_image": (time.perf_counter() - t0) / count, "images": count}
        mp = 1024
        phi = synth.make_phi(c.m, c.N, st, rows=(0, mp))
        x = synth.make_images(c.n, 0, 1, c.n_blobs, c.n_rects, c.texture_var)
        y = synth.measure(phi, x, st)
        params = synth.make_params().rounded(st)
        t0 = time.perf_counter()
        oracle.proxy(phi, y)
        t_rows = time.perf_counter() - t0
        small = phi[:64]
        t0 = time.perf_counter()
        oracle.forward(y[:, :64], small, params, c.n, c.n, threads=1)
        t_fwd = time.perf_counter() - t0
        return name, {"s_per_image": t_fwd + t_rows * (c.m - 64) / mp, "images": 1,
                      "extrapolated": f"proxy timed on {mp} of {c.m} rows (linear in M)"}

    jobs = [("tiny", 4), ("paper", 16), ("lowrate", 16), ("larger", 4), ("stress", 1)]
    with ThreadPoolExecutor(len(jobs)) as ex:
        return dict(ex.map(lambda j: one(*j), jobs))


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="lowrate", choices=["tiny", "paper", "lowrate", "larger", "stress"])
    ap.add_argument("--batch", type=int, default=0, help="override the per-GPU batch (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle time for cpu_baseline")
    ap.add_argument("--no-cpu-configs", action="store_true", help="skip the per-config single-thread oracle times")
    ap.add_argument("--no-oracle-check", action="store_true", help="output check: bitwise part only")
    ap.add_argument("--no-check", action="store_true", help="skip the output check (profiling runs: launch lists)")
    ap.add_argument("--no-train", action="store_true", help="skip the training-step probe")
    ap.add_argument("--no-sustained", action="store_true", help="skip the 2-s sustained (power-capped) run")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: --warmup < 3 breaks the timing rules", file=sys.stderr)
    if args.gpus < 1:
        print("--gpus must be >= 1", file=sys.stderr)
        return 2
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N`: start N ranks (one process per GPU) under torchrun; rank 0 prints the line
        return subprocess.call(launcher_cmd(sys.argv[1:] if argv is None else list(argv), args.gpus, free_port()))
    _, world, _ = dist_env()
    if world != args.gpus:
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
