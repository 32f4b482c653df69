#!/usr/bin/env python
"""Benchmark: EC / surface-area / volume curves of a 3D float32 Gaussian
random field (BASELINE.json configs[4]: 2048^3, sigma = 4 voxels, 512 levels,
z-slab partitioned over N GPUs with one NCCL all-reduce of the histograms).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

One step = one pass of the hot path over the whole field: the fused quantize +
line-decomposition histogram kernel (ft_lines3d) on this rank's z-slab (+2
halo planes), NCCL all-reduce of the histogram (N > 1), device scan into the
three curves.  ``value`` is whole-job Gvoxels/s with the field resident in HBM
(max over ranks of the CUDA-event time); ``e2e`` is the same through the public
API (``descriptor_curves`` on an ``ArraySource`` over PINNED HOST memory:
chunked H2D overlapped with the kernel, curves read back to the host).
``--impl reference`` times the reference algorithm on the host CPU cores (the
C restatement in oracle/, all threads) on a bounded sample of the same field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (shape, sigma, M, dtype, descriptors)
    "c5": ((2048, 2048, 2048), 4.0, 511, "f32", ("ec", "surface-area", "volume")),
    "c4a": ((512, 512, 512), 3.0, 255, "f32", ("ec", "surface-area", "volume")),
    "small": ((256, 256, 256), 3.0, 255, "f32", ("ec", "surface-area", "volume")),
}


NCU_C5 = "profiles/r02/s5/evidence/lines3d_c5.summary.txt"  # latest ncu --set full capture of the C5 kernel


def ncu_traffic(path=ROOT / NCU_C5):
    """DRAM bytes (read + write) per launch of the main kernel from the committed
    ncu --set full summary (None when absent)."""
    try:
        vals = {}
        for line in path.read_text().splitlines():
            parts = line.split()
            if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[parts[2]]
                vals[parts[0]] = float(parts[1]) * scale
        return int(sum(vals.values())) if len(vals) == 2 else None
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed
    region: NVML polled every 5 ms on a thread (nvidia-smi -lms 100 when NVML
    is unavailable)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index, uuid=None, period_s=0.005):
        self.index, self.uuid, self.period = index, uuid, period_s
        self.rows = []      # (sm_mhz, max_mhz, power_w, {reason names})
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        h = None
        if self.uuid:
            try:
                h = pynvml.nvmlDeviceGetHandleByUUID(self.uuid)
            except pynvml.NVMLError:
                h = None
        if h is None:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        return pynvml, h

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001 -- NVML missing or unusable: fall back
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), pw, {n for n, b in bits.items() if r & b}))
            except nv.NVMLError:
                pass
            time.sleep(self.period)

    def _read(self):
        for line in self.proc.stdout:
            r = [c.strip() for c in line.split(",")]
            try:
                self.rows.append((float(r[1]), float(r[2]), float(r[3]),
                                  {n for n, v in zip(self.NAMES, r[5:9]) if v.lower() == "active"}))
            except (IndexError, ValueError):
                pass

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.nvml:
            self.thread.join(timeout=1)
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "power_w_max": round(max(r[2] for r in self.rows), 1),
                "reasons": sorted(set().union(*(r[3] for r in self.rows))), "samples": len(self.rows),
                "source": "nvml 5 ms" if self.nvml else "nvidia-smi 100 ms"}


def _gpu_uuid(dev):
    import torch
    try:
        return "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001
        return None


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference(x_host, M, lo_hi, descs, budget_s=15.0, threads=None):
    """Oracle (C restatement of the reference gather, all host threads) on a
    bounded slab sample of the field; returns (Gvoxels/s, cells, seconds, threads)."""
    from oracle import oracle
    threads = threads or os.cpu_count() or 1
    H, W, D = x_host.shape
    tables = [oracle.BUILTIN_3D[(d, "26C" if d == "ec" else None)] for d in descs]

    last = [None]

    def run(nplanes):
        sample = np.ascontiguousarray(x_host[:nplanes])
        t0 = time.perf_counter()
        q_in, q_out = oracle.gather3d(sample, M, value_range=lo_hi, workers=threads, rows=(0, nplanes))
        for w in tables:
            oracle.descriptor_numerators(q_in, q_out, M, w)
        dt = time.perf_counter() - t0
        last[0] = (q_in, q_out)
        return dt

    # the oracle splits vertex rows over threads like the reference
    # (_parallel.py:8-24): keep >= 4 planes per thread so all cores work
    n = min(H, 4 * threads)
    t = run(n)
    while t < 0.5 and n < H:
        n = min(H, n * 2)
        t = run(n)
    n_final = max(min(H, 4 * threads), min(H, int(n * budget_s / max(t, 1e-6))))
    # the reference split hands the remainder rows to the LAST worker
    # (_parallel.py:19-23): a sample that is a multiple of the thread count
    # keeps its threads evenly loaded (110 rows on 16 threads would leave 20
    # to the last one and time the reference ~3x too slow)
    n_final = max(threads, n_final - n_final % threads) if n_final > threads else n_final
    t, maps = run(n_final), last[0]
    cells = n_final * W * D
    return cells / t / 1e9, cells, t, threads, n_final, maps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + ["c5s"], default="c5",
                    help="c5s: the 4096^3 f32 (256 GiB) instance through the chunk-streaming path")
    ap.add_argument("--seed", type=int, default=2311)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--kernel", choices=("lines", "lattice"), default="lines",
                    help="fused curve kernel (A/B): ft_lines3d (default) or ft_lattice3d")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: plumbing check with several ranks sharing one GPU (no performance claim)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: W >= 3 is the contract; raising warmup to 3", file=sys.stderr)
        args.warmup = 3

    import torch
    ws, rank, local = dist_env()
    if args.config == "c5s":
        if rank == 0:
            (run_reference_c5s if args.impl == "reference" else run_c5s)(args)
        return
    shape, sigma, M, _, descs = CONFIGS[args.config]
    H, W, D = shape
    config = {"workload": f"{args.config}: 3D float32 smoothed Gaussian random field {H}x{W}x{D}, "
                          f"sigma={sigma:g} voxels, min-max normalised, {M + 1} levels; "
                          f"curves: {', '.join(descs)}",
              "field": [H, W, D], "sigma": sigma, "levels": M + 1, "descriptors": list(descs),
              "partition": f"z-slabs over {ws} rank(s), 2 low halo planes" +
                           (f", {args.dist_backend} all-reduce" if ws > 1 else ""),
              "l2": "inputs larger than L2 (field >> 126 MB)"}

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, shape, sigma, M, descs, config, ws)
        return

    import paper_2311_11740_b200 as ft
    from paper_2311_11740_b200 import engine, synth
    from paper_2311_11740_b200._parallel import held_rows, split_blocks

    # one GPU per rank; the gloo plumbing check may put several ranks on one GPU
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    blocks = split_blocks(H + 1, ws)
    a, b = blocks[rank] if rank < len(blocks) else (H + 1, H + 1)
    r0, r1 = held_rows(a, b, H)

    # ---- field (setup, untimed) -------------------------------------------
    x = synth.grf_slab(shape, sigma, args.seed, (r0, r1), dev)
    mn, mx = x.min(), x.max()
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    synth.normalise_(x, mn, mx)
    torch.cuda.synchronize()

    quant = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
    tables = [ft.builtin_weights(d, "26C") for d in descs]
    eighths = [t.eighths for t in tables]
    plan = ft.lattice.fused_plan(3, eighths, lines_ok=args.kernel == "lines" and engine.lines_ok(M))
    kind = ft.gather.Kind(plan[0], plan[1])
    row_w = plan[2]
    kname = {"lines": "lines3d_kernel (line-decomposition EC / surface / volume histograms)",
             "lattice": "lattice3d_rb_kernel (element min-filter histograms)"}[plan[0]]
    hist = kind.new(3, M, dev)
    stream = torch.cuda.current_stream(dev)
    k_start, k_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(ev=None):
        # the fused curve path: level histograms (ft_lines3d) -> NCCL
        # all-reduce (N > 1) -> device prefix scan into the three curves;
        # ev = (start, end) events around the histogram kernel
        hist.zero_()
        if ev is not None:
            ev[0].record(stream)
        kind.launch(3, x, shape, M, quant, (a, b), first=r0, hist=hist)
        if ev is not None:
            ev[1].record(stream)
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(hist)
        return engine.curves_from_rows(hist, M, row_w)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the dominant kernel's launch durations, measured inside the timed region
    # (event pairs on the launching stream around every ft_lines3d launch)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index, _gpu_uuid(dev)) as clk:
        t0.record(stream)
        for i in range(args.steps):
            step(kev[i])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1) / args.steps
    kernel_ms = [e0.elapsed_time(e1) for e0, e1 in kev]
    kms = statistics.mean(kernel_ms)
    t_ms = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms, kms = t_ms.tolist()
    cells = H * W * D
    value = cells / (ms / 1e3) / 1e9
    # full-size parity properties (no oracle can run 2048^3 here): the curves
    # of the benchmark kernel, of the independent drop-in map kernel on the
    # same field, and (below) of the streamed end-to-end path must agree bit
    # for bit; and the whole box (level M) is one contractible solid
    resident = step().cpu().numpy() // plan[3][:, None]
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    # the contribution-map kernel (drop-in gather_3d_*), same field, reported beside
    mhist = engine.new_hist(3, M, dev)
    map_ms = []
    for _ in range(3):
        mhist.zero_()
        k_start.record(stream)
        engine.launch_hist(3, x, shape, M, quant, rows=(a, b), first=r0, hist=mhist)
        k_end.record(stream)
        torch.cuda.synchronize()
        map_ms.append(k_start.elapsed_time(k_end))
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(mhist)
    _, _, map_num = engine.finalize(3, M, mhist, maps=False, tables=eighths)
    map_curves = map_num.cpu().numpy()
    del mhist
    map_gvox = (r1 - r0) * W * D / (statistics.median(map_ms) / 1e3) / 1e9

    # ---- end to end through the public API, host-resident input ----------
    e2e = None
    if not args.no_e2e:
        e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
        host = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(x)
        del x
        torch.cuda.empty_cache()
        src = ft.ArraySource(host, M, value_range=(0.0, 1.0))  # pinned: H2D straight from its pages
        e_times = []
        for it in range(1 + e2e_steps):
            barrier()
            torch.cuda.synchronize()
            s = time.perf_counter()
            if ws == 1:
                # the public call a user makes
                curves = np.stack([c.numerators for c in ft.descriptor_curves(src, tables, device=dev,
                                                                              chunk_bytes=512 << 20)])
            else:
                # the rank's planes [r0, r1) stand for global planes
                h = ft.gather.stream_hist(_ShiftedSource(src, r0, H), 3, dev, (a, b), chunk_bytes=512 << 20,
                                          kind=kind)
                import torch.distributed as dist
                dist.all_reduce(h)
                curves = engine.curves_from_rows(h, M, row_w).cpu().numpy() // plan[3][:, None]
            torch.cuda.synchronize()
            if it:
                e_times.append(time.perf_counter() - s)
        et = torch.tensor([statistics.mean(e_times)], dtype=torch.float64, device=dev)
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": round(cells / et.item() / 1e9, 4), "unit": "Gvoxels/s",
               "h2d_bytes_per_step": int((r1 - r0) * W * D * 4 * ws), "d2h_bytes_per_step": int(curves.nbytes),
               "path": ("fieldtopo.descriptor_curves(ArraySource(pinned host tensor), tables) -- the public call"
                        if ws == 1 else "per rank: gather.stream_hist over its planes + NCCL all-reduce")
                       + "; 512 MiB chunks, double-buffered H2D overlapped with the kernel, curves to host"}
        x = None
    box = {"ec": 8, "surface-area": 8 * 2 * (H * W + W * D + H * D), "volume": 8 * H * W * D}
    checks = {"map_kernel_curves_equal": bool(np.array_equal(map_curves, resident)),
              "e2e_curves_equal": None if e2e is None else bool(np.array_equal(curves, resident)),
              "full_box_at_level_M": bool(all(int(resident[i][M]) == box[d] for i, d in enumerate(descs))),
              "volume_monotone": bool(np.all(np.diff(resident[list(descs).index("volume")]) >= 0))}

    # ---- CPU baseline (rank 0, N = 1 only) ----------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        xs = host.numpy() if e2e is not None else x.cpu().numpy()
        v, n, secs, thr, nplanes, (oq_in, oq_out) = cpu_reference(xs, M, (0.0, 1.0), descs, args.cpu_budget)
        cpu = {"value": round(v, 6), "unit": "Gvoxels/s", "cores": thr, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{n // (W * D)} planes x {W}x{D} of the same field ({n} voxels, {secs:.1f} s), "
                         "oracle/ft_oracle.c gather + curves"}
        # parity on the sample: the drop-in map kernel on the same planes and
        # vertex rows [0, nplanes) must equal the oracle's maps bit for bit
        xd = engine.to_device(xs[:nplanes], dev)
        sh = engine.launch_hist(3, xd, (nplanes, W, D), M, quant, rows=(0, nplanes))
        sq_in, sq_out, _ = engine.finalize(3, M, sh, maps=True)
        checks["oracle_sample_maps_equal"] = bool(np.array_equal(engine.as_uint64(sq_in), oq_in)
                                                  and np.array_equal(engine.as_uint64(sq_out), oq_out))
        checks["oracle_sample"] = f"vertex rows [0, {nplanes}) of the benchmark field"
        del xd, sh

    if rank == 0:
        peak, peak_kind = peaks()
        # algorithmic bytes: every cell of the rank's planes read once (f32)
        bytes_per_launch = (r1 - r0) * W * D * 4
        achieved = bytes_per_launch / (kms / 1e3) / 1e9
        out = {"metric": "Gvoxels/s for EC curve (1/2/4/8 B200) and % of HBM roofline vs CPU ref",
               "value": round(value, 4), "unit": "Gvoxels/s", "n_gpus": ws, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32 in, int32 levels, u64 histograms",
               "data": "synthetic (seeded device-generated GRF; no dataset in the reference)",
               "config": config, "checks": checks,
               "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                            "frac": round(achieved / peak, 4),
                            "traffic": ncu_traffic() if plan[0] == "lines" and (H, W, D) == (2048, 2048, 2048) else None,
                            "traffic_source": NCU_C5 + " (ncu --set full, one launch, "
                                              "dram__bytes_read + dram__bytes_write)",
                            "kernel": kname + ", mean launch duration over the timed region (CUDA events on the launching stream)",
                            "kernel_ms": round(kms, 4), "peak_source": peak_kind,
                            "algorithmic_bytes_per_launch": int(bytes_per_launch)},
               "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": 2 * args.steps,
               "map_path": {"kernel": "hist3d_march (transition-class maps, gather_3d_*)",
                            "value": round(map_gvox, 4), "unit": "Gvoxels/s",
                            "kernel_ms": round(statistics.median(map_ms), 4)},
               "clocks": clk.summary()}
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


class _ShiftedSource:
    """Present a host array holding global planes [r0, r0 + n) as the full
    field (reads only ever touch the rank's planes)."""

    mode = "file-backed"

    def __init__(self, src, r0, H):
        self.src, self.r0, self.H = src, r0, H
        self.ndim, self.max_level, self.quant, self.dtype = 3, src.max_level, src.quant, src.dtype
        self.height, self.width, self.depth = H, src.width, src.depth
        self.shape = (H, src.width, src.depth)
        self.peak_field_bytes = 0
        self.parallel_reads = True
        self.pinned_window = (lambda a, b: src.pinned_window(a - r0, b - r0)) if src.pinned_window else None

    def note_resident(self, n):
        self.peak_field_bytes = max(self.peak_field_bytes, n)

    def read_rows(self, a, b, out):
        self.src.read_rows(a - self.r0, b - self.r0, out)


def run_reference(args, shape, sigma, M, descs, config, ws):
    """CPU baseline arm: the reference algorithm (oracle/ft_oracle.c, a C
    restatement of fieldtopo's Numba kernels) on all host cores."""
    import torch
    from paper_2311_11740_b200 import synth
    H, W, D = shape
    # same field bytes as our arm: generate on the GPU if present, else a CPU
    # stand-in of the same distribution; only a bounded slab is needed
    nplanes = min(H, max(64, 8 * (os.cpu_count() or 1)))
    if torch.cuda.is_available():
        x = synth.grf_slab(shape, sigma, args.seed, (0, nplanes), torch.device("cuda", 0))
        x = ((x - x.min()) / (x.max() - x.min())).cpu().numpy()
    else:
        x = np.random.default_rng(args.seed).random((nplanes, W, D), dtype=np.float32)
    times = []
    for it in range(args.warmup + args.steps):
        v, n, secs, thr, _, _ = cpu_reference(x, M, (0.0, 1.0), descs, budget_s=max(2.0, args.cpu_budget / 3))
        if it >= args.warmup:
            times.append(v)
    v = statistics.mean(times)
    out = {"impl": "reference", "metric": "Gvoxels/s for EC curve (1/2/4/8 B200) and % of HBM roofline vs CPU ref",
           "value": round(v, 6), "unit": "Gvoxels/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 in, int64 levels",
           "data": "synthetic (same seeded GRF slab)", "config": config,
           "cpu_baseline": {"value": round(v, 6), "unit": "Gvoxels/s", "cores": thr, "kind": "port",
                            "cpu_model": cpu_model(), "sample": f"{n // (W * D)} planes x {W}x{D} per step (bounded sample)"},
           "e2e": {"value": round(v, 6), "unit": "Gvoxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


C5S = dict(shape=(4096, 4096, 4096), period=64, sigma=4.0, M=511, descs=("ec", "surface-area", "volume"))


def _c5s_config():
    H, W, D = C5S["shape"]
    return {"workload": f"c5s: 3D float32 smoothed Gaussian random field {H}x{W}x{D} (256 GiB, larger than "
                        f"HBM and than this host's RAM), sigma={C5S['sigma']:g} voxels, {C5S['M'] + 1} levels, "
                        "through the low-memory chunk-streaming path; curves: " + ", ".join(C5S["descs"]),
            "field": [H, W, D], "sigma": C5S["sigma"], "levels": C5S["M"] + 1, "descriptors": list(C5S["descs"]),
            "source": f"plane-periodic field (period {C5S['period']} planes, a GRF periodic along i) served "
                      f"from a pinned ring of {2 * C5S['period']} planes ({2 * C5S['period'] * W * D * 4 >> 30} GiB)",
            "l2": "inputs larger than L2 (field >> 126 MB)"}


def _c5s_base(args, dev):
    import torch
    from paper_2311_11740_b200 import synth
    H, W, D = C5S["shape"]
    P = C5S["period"]
    base = synth.grf_slab((P, W, D), C5S["sigma"], args.seed, (0, P), dev)
    synth.normalise_(base, base.min(), base.max())
    return base


def run_c5s(args):
    """C5s: 4096^3 float32 (256 GiB) through the chunk-streaming engine
    (BASELINE.json configs[4]'s low-memory instance).  Every plane crosses
    PCIe once (pinned ring -> two device buffers, halo planes carried
    device-to-device); the line kernel runs on each chunk as it lands."""
    import torch
    import paper_2311_11740_b200 as ft
    from paper_2311_11740_b200 import engine, synth
    from paper_2311_11740_b200._parallel import held_rows, split_blocks
    from oracle import oracle
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    H, W, D = C5S["shape"]
    P, M = C5S["period"], C5S["M"]
    base = _c5s_base(args, dev)
    ring = torch.empty((2 * P, W, D), dtype=torch.float32, pin_memory=True)
    ring[:P].copy_(base)
    ring[P:].copy_(ring[:P])
    src = synth.PeriodicPlanes(ring, H, M, (0.0, 1.0))
    tables = [ft.builtin_weights(d, "26C") for d in C5S["descs"]]
    plane_bytes = W * D * 4
    chunk_bytes = 32 * plane_bytes  # 2 GiB windows (<= the ring period)

    # measured pinned host -> device copy peak (the PCIe ceiling of this path)
    hbuf = ring[:32].reshape(-1)
    dbuf = torch.empty_like(hbuf, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d = []
    for _ in range(6):
        e0.record()
        dbuf.copy_(hbuf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d.append(hbuf.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del dbuf
    h2d_peak = max(h2d[1:])

    steps = max(1, min(args.steps, 2))
    times = []
    with ClockSampler(0) as clk:
        for it in range(1 + steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            curves = np.stack([c.numerators for c in ft.descriptor_curves(src, tables, device=dev,
                                                                          chunk_bytes=chunk_bytes)])
            torch.cuda.synchronize()
            if it:
                times.append(time.perf_counter() - t0)
    secs = statistics.mean(times)
    cells = H * W * D
    value = cells / secs / 1e9
    gbs = cells * 4 / secs / 1e9

    # checks: the same field device-resident slab by slab (no streaming engine)
    plan = ft.lattice.fused_plan(3, [t.eighths for t in tables], lines_ok=True)
    dring = ring.to(dev)
    hist = engine.new_lines_hist(M, dev)
    for a, b in split_blocks(H + 1, cdiv_int(H + 1, P - 2)):
        r0, r1 = held_rows(a, b, H)
        s0 = r0 % P
        engine.launch_lines(dring[s0:s0 + (r1 - r0)], (H, W, D), M, src.quant, rows=(a, b), first=r0, hist=hist)
    resident = engine.curves_from_rows(hist, M, plan[2]).cpu().numpy() // plan[3][:, None]
    del dring, hist
    # the oracle on vertex rows [0, n) of the field vs the drop-in map kernel
    n = 24
    q_in, q_out = oracle.gather3d(ring[:n].numpy(), M, value_range=(0.0, 1.0), workers=os.cpu_count(), rows=(0, n))
    mh = engine.launch_hist(3, base[:n].contiguous(), (n, W, D), M, src.quant, rows=(0, n))
    mq_in, mq_out, _ = engine.finalize(3, M, mh, maps=True)
    box = {"ec": 8, "surface-area": 8 * 2 * (H * W + W * D + H * D), "volume": 8 * H * W * D}
    descs = list(C5S["descs"])
    checks = {"resident_slabs_curves_equal": bool(np.array_equal(curves, resident)),
              "full_box_at_level_M": bool(all(int(curves[i][M]) == box[d] for i, d in enumerate(descs))),
              "volume_monotone": bool(np.all(np.diff(curves[descs.index("volume")]) >= 0)),
              "oracle_sample_maps_equal": bool(np.array_equal(engine.as_uint64(mq_in), q_in)
                                               and np.array_equal(engine.as_uint64(mq_out), q_out)),
              "oracle_sample": f"vertex rows [0, {n}) of the field"}
    out = {"metric": "Gvoxels/s for EC curve (1/2/4/8 B200) and % of HBM roofline vs CPU ref",
           "value": round(value, 4), "unit": "Gvoxels/s", "n_gpus": 1, "steps": steps, "warmup": 1,
           "ms_per_step": round(secs * 1e3, 2), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f32 in, int32 levels, u64 histograms", "data": "synthetic (seeded device-generated GRF)",
           "config": _c5s_config(), "checks": checks,
           "roofline": {"bound": "pcie-h2d", "achieved": round(gbs, 2), "peak": round(h2d_peak, 2), "unit": "GB/s",
                        "frac": round(gbs / h2d_peak, 4), "traffic": None,
                        "peak_source": "measured in this run: pinned 2 GiB host->device copy, best of 5 "
                                       "(CUDA events)",
                        "h2d_bytes_per_step": cells * 4},
           "e2e": {"value": round(value, 4), "unit": "Gvoxels/s", "h2d_bytes_per_step": cells * 4,
                   "d2h_bytes_per_step": int(curves.nbytes),
                   "path": "descriptor_curves(PeriodicPlanes) -- pinned ring -> 2 GiB device windows, double-"
                           "buffered H2D on a side stream overlapped with ft_lines3d, halo planes carried D2D"},
           "gpu_launches": None, "clocks": clk.summary()}
    print(json.dumps(out))


def cdiv_int(a, b):
    return -(-a // b)


def run_reference_c5s(args):
    """CPU reference arm for c5s: the oracle on a bounded sample (the first
    planes of the same periodic field), all host cores."""
    import torch
    H, W, D = C5S["shape"]
    M = C5S["M"]
    base = _c5s_base(args, torch.device("cuda", 0)) if torch.cuda.is_available() else \
        np.random.default_rng(args.seed).random((C5S["period"], W, D), dtype=np.float32)
    x = base.cpu().numpy() if hasattr(base, "cpu") else base
    v, n, secs, thr, _, _ = cpu_reference(x, M, (0.0, 1.0), C5S["descs"], budget_s=max(2.0, args.cpu_budget / 3))
    out = {"impl": "reference", "metric": "Gvoxels/s for EC curve (1/2/4/8 B200) and % of HBM roofline vs CPU ref",
           "value": round(v, 6), "unit": "Gvoxels/s", "n_gpus": 1, "steps": 1, "warmup": 0,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 in, int64 levels",
           "data": "synthetic (same periodic GRF base)", "config": _c5s_config(),
           "cpu_baseline": {"value": round(v, 6), "unit": "Gvoxels/s", "cores": thr, "kind": "port",
                            "cpu_model": cpu_model(), "sample": f"{n // (W * D)} planes x {W}x{D} (bounded sample)"},
           "e2e": {"value": round(v, 6), "unit": "Gvoxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
