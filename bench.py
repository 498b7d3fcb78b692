"""bench.py — GNP hot path on B200 (driver contract: one JSON line on rank 0).

metric (both arms, BASELINE.json's own string): "GNP M·v applies/sec +
fused-layer HBM GB/s vs peak; FGMRES solve time"; unit applies/s.

Headline workload (default): C5 = BASELINE configs[4], the largest
single-GPU config and one of the two the >= 60 %-of-HBM target is stated on:
2D anisotropic diffusion 2048^2, 9-point (n = 4,194,304, nnz = 37,724,164),
Â = A/γ in fp32, GNP d = 32, hidden 32, 8 Res-GCONV layers, Xavier-uniform
weights from seed 0.  One step = one M·v apply of a fresh right-hand side.
  value  : device-resident fp32 inputs (gnpc_apply_device_f32), CUDA events per
           step on the launching stream; L2 flushed (512 MiB write) between
           steps (C5's 12 GB working set exceeds L2 anyway).
  e2e    : the reference-facing C-ABI call gnpc_apply with pinned HOST f64
           buffers: b host->device and M(b) device->host inside every step.
  roofline: the dominant kernel (k_layer_sell<32>, one fused Res-GCONV layer
           per launch), bytes = 4(n+1) + 8 nnz + 8 n d per launch (SURVEY §8d,
           DESIGN.md §4), time = its average launch duration from CUDA events
           around every launch on the launching stream (gnpc_apply_profile).
  fgmres : one device FGMRES solve of the config (restart/rtol per BASELINE)
           with SURVEY §8d's per-iteration byte model and its GB/s.
  cpu_baseline: the unmodified reference gnn_apply (oracle/_ref), 1 thread,
           on a bounded sample (the same generator at a smaller size, work
           scaled by the row ratio — every cost of the apply is O(n + nnz)).
  configs: the other north-star configs measured in the same run — C4 (n = 2^20
           power-law, d = 16), C2 (3D conv-diff 64^3, d = 16) and C3 (training,
           steps/s) — each with its own roofline.
--config c1|c2|c3|c4|c5 prints that config's line alone.
--impl reference: the reference CPU implementation (oracle/_ref; imports only
           oracle/), all usable host threads, same metric/config/unit.
N > 1 (torchrun): apply = independent replicas (value = Σ applies / max-rank
time); C3 = data-parallel over samples with an NCCL gradient all-reduce.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _baseline_metric():
    try:
        return json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    except Exception:
        return "GNP M·v applies/sec + fused-layer HBM GB/s vs peak; FGMRES solve time"


METRIC = _baseline_metric()

# name: generator (kind, size, p0, p1, seed), dims, rhs (kind, seed), fgmres
# (restart, rtol, maxiters), description, bounded CPU sample (size, row ratio)
CONFIGS = {
    "c1": dict(gen=("convection_diffusion", 64, 0.0, 0.0, 0), dims=(16, 32, 8), rhs=("gauss", 1),
               fg=(10, 1e-8, 100), desc="C1 2D 5-pt Laplacian 64x64 (n=4096), GNP d=16 L=8",
               sample=(64, 1)),
    "c2": dict(gen=("c2_convdiff3d", 64, 10.0, 0.0, 0), dims=(16, 32, 8), rhs=("Ax", 1),
               fg=(30, 1e-6, 100), desc="C2 3D conv-diff 7-pt upwind 64^3 Pe=10 (n=262144), GNP d=16 L=8",
               sample=(64, 1)),
    "c4": dict(gen=("c4_powerlaw", 1 << 20, 2.2, 0.0, 4), dims=(16, 32, 8), rhs=("gauss", 4),
               fg=(30, 1e-6, 100),
               desc="C4 power-law random n=2^20 (alpha 2.2, rows 4..2048), GNP d=16 L=8",
               sample=(1 << 18, 4)),
    "c5": dict(gen=("c5_aniso9pt", 2048, 1e-3, 30.0, 0), dims=(32, 32, 8), rhs=("Ax", 3),
               fg=(50, 1e-6, 100), desc="C5 2D anisotropic 9-pt 2048^2 (eps 1e-3, 30deg), GNP d=32 L=8",
               sample=(512, 16)),
}
C3 = dict(gen=("c3_varcoeff2d", 512, 2.0, 0.0, 2), dims=(32, 32, 8), batch=32, monitor=16,
          desc="C3 2D var-coeff diffusion 512^2 lognormal(0,2^2), d=32 L=8 B=32, Adam 1e-3",
          sample=(256, 4))
C3_METRIC = "GNP training steps/s (C3)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a thread, nvidia-smi -lms 100 as the
    fallback."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, sm_max_mhz, set(reasons))
        self.stop_ev = threading.Event()
        self.t = None
        self.proc = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                    "hw_power_brake_slowdown": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), {k for k, v in bits.items() if r & v}))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return

        def reader():
            for line in self.proc.stdout:
                r = [x.strip() for x in line.split(",")]
                try:
                    self.rows.append((float(r[0]), float(r[1]),
                                      {nm for nm, v in zip(names, r[2:6]) if v.lower() == "active"}))
                except (ValueError, IndexError):
                    continue

        self.t = threading.Thread(target=reader, daemon=True)
        self.t.start()

    def stop(self):
        self.stop_ev.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.t is not None:
            self.t.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0}
        reasons = set()
        for r in self.rows:
            reasons |= r[2]
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": sorted(reasons),
                "samples": len(self.rows)}


# --------------------------------------------------------------- byte models
def a_bytes(n, nnz):
    return 4 * (n + 1) + 8 * nnz


def layer_bytes(n, nnz, d):
    """one fused Res-GCONV layer reads Â and X once, writes Y once."""
    return a_bytes(n, nnz) + 8 * n * d


def apply_bytes(n, nnz, d, L):
    return 12 * n + 8 * n * d + L * layer_bytes(n, nnz, d)


def fgmres_bytes(n, nnz, d, L, iters, restart, reorth_steps):
    """SURVEY §8d FGMRES byte model: per Arnoldi step j (0-based in its cycle)
    the apply, v read (fp64), w = A z, MGS 40n(j+1) (+ again when the
    re-orthogonalisation pass is taken), two norms, normalise, store z; per
    cycle x += Z y and the true residual; plus the initial residual.  The
    device counts re-orth passes but not their positions: they are charged at
    the mean basis length of the solve."""
    A = a_bytes(n, nnz)
    ab = apply_bytes(n, nnz, d, L) if L else 4 * n
    tot, mgs = A + 24 * n, 0
    js = [s % restart for s in range(iters)]
    for j in js:
        tot += ab + 4 * n + A + 12 * n + 40 * n * (j + 1) + 16 * n + 16 * n + 4 * n
        mgs += 40 * n * (j + 1)
    if iters:
        tot += reorth_steps * mgs / iters
    cycles = -(-iters // restart) if iters else 0
    for c in range(cycles):
        k = min(restart, iters - c * restart)
        tot += 4 * n * k + 16 * n + A + 24 * n
    return int(tot)


def train_step_bytes(n, nnz, d, B, L):
    """SURVEY §8(d) canonical algorithmic bytes of one training step."""
    A = a_bytes(n, nnz)
    T = 4 * n * B * d
    fwd = L * (A + 3 * T)
    bwd = L * (A + 5 * T)
    enc = (T + 4 * n * B) * 2
    dec = (T + 4 * n * B) + (2 * T + 4 * n * B)
    loss = 2 * A + 16 * n * B
    return fwd + bwd + enc + dec + loss


def monitor_bytes(n, nnz, d, MB, L):
    """forward of the fixed monitoring batch + its loss (no gradient)."""
    A = a_bytes(n, nnz)
    T = 4 * n * MB * d
    return L * (A + 2 * T) + (T + 4 * n * MB) * 2 + A + 16 * n * MB


def pair_bytes(n, nnz, B):
    """SURVEY §8d pair generation: write x (f64) + b = A x (f64 values)."""
    return 8 * n * B + 4 * (n + 1) + 16 * nnz + 16 * n * B


def dp_of(d):
    return 4 if d <= 4 else (8 if d <= 8 else (16 if d <= 16 else (32 if d <= 32 else 64)))


# --------------------------------------------------------------- reference side
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    return oracle


def ref_matrix(gen, size=None):
    """The config matrix built by the oracle's restatement of the generator
    (test infrastructure; no product code), prescaled by γ, values rounded to
    fp32 like the device copy, as f64."""
    oracle = _oracle()
    o = oracle.restatement()
    kind, sz, p0, p1, seed = gen
    sz = size or sz
    a = o.gen_convection_diffusion(sz, p0) if kind == "convection_diffusion" else o.gen_named(kind, sz, p0, p1, seed)
    return o.prescale(a, o.gershgorin_gamma(a)).rounded_f32()


def ref_impl():
    oracle = _oracle()
    if oracle.reference_available():
        return oracle.reference(), "reference"
    return oracle.restatement(), "port"


def _ref_threads(per_call_bytes):
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    return max(1, min(os.cpu_count() or 1, int(avail * 0.6 // max(per_call_bytes, 1))))


def ref_apply_sampler(cfg_name, threads=None):
    """One 'step' of the reference apply arm: `threads` concurrent reference
    gnn_apply calls on the config's generator at the sample size; returns
    (run_step() -> seconds, full-size applies per step, description)."""
    cfg = CONFIGS[cfg_name]
    size, ratio = cfg["sample"]
    a = ref_matrix(cfg["gen"], size)
    impl, kind = ref_impl()
    d, h, L = cfg["dims"]
    p = impl.init_params(d, h, L, 0).astype(np.float32).astype(np.float64)
    b = impl.gaussian_vector(cfg["rhs"][1], a.n)
    cache = 8 * a.n * ((3 * L + 1) * d + 4 * h + 4)  # the reference keeps its ForwardCache
    T = threads or _ref_threads(cache)

    def one():
        if kind == "reference":
            impl.time_gnn_apply(a, (d, h, L), p, b, 1)
        else:
            impl.gnn_apply(a, (d, h, L), p, b)

    def run():
        t0 = time.perf_counter()
        ts = [threading.Thread(target=one) for _ in range(T)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    where = "the full-size matrix" if ratio == 1 else \
        f"the same generator at size {size} (n={a.n}, nnz={a.nnz}; 1/{ratio} of the rows, scaled by {ratio})"
    desc = f"{T} concurrent reference gnn_apply call(s) per step on {where}, fp32-rounded inputs as f64"
    return run, T / ratio, desc, kind, T


def ref_train_sampler(threads=None):
    """One 'step' of the reference training arm: `threads` concurrent
    reference forward + L1 loss + backward calls, one column each
    (src/gnn.cpp:426-438 runs its columns over hardware_concurrency() threads),
    on the C3 generator at the sample size; full C3 steps per sample =
    threads / (B * row ratio)."""
    size, ratio = C3["sample"]
    a = ref_matrix(C3["gen"], size)
    impl, kind = ref_impl()
    dims = C3["dims"]
    p = impl.init_params(*dims, 0).astype(np.float32).astype(np.float64)
    x = impl.gaussian_vector(5, a.n)
    b = impl.spmv(a, x)
    d, h, L = dims
    cache = 8 * a.n * ((3 * L + 1) * d + 4 * h + 8 * d)
    T = threads or _ref_threads(cache)

    def one():
        impl.batch_loss_grads(a, dims, p, x, b, 1)

    def run():
        t0 = time.perf_counter()
        ts = [threading.Thread(target=one) for _ in range(T)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    desc = (f"{T} concurrent reference forward+loss+backward column(s) per step on the C3 generator at "
            f"{size}^2 (n={a.n}; 1/{ratio} of the rows); one C3 step = {C3['batch']} columns at 512^2")
    return run, T / (C3["batch"] * ratio), desc, kind, T


REF_BUDGET_S = 150.0  # bound on the reference arm's timed loop (seconds)


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    the unmodified reference library) on all usable host threads; imports
    only oracle/ (no product code).  Rank 0 alone runs it."""
    if rank != 0:
        print(json.dumps({"impl": "reference", "rank": rank, "skipped": "rank 0 only"}), file=sys.stderr)
        return
    cfg_name = args.config
    if cfg_name == "c3":
        run, units, desc, kind, T = ref_train_sampler()
        metric, unit, wl = C3_METRIC, "steps/s", C3["desc"]
        dims = C3["dims"]
    else:
        run, units, desc, kind, T = ref_apply_sampler(cfg_name)
        metric, unit, wl = METRIC, "applies/s", CONFIGS[cfg_name]["desc"]
        dims = CONFIGS[cfg_name]["dims"]
    # a step is bounded (seconds); warm-up stops after REF_BUDGET_S / 6 and the
    # timed loop runs as many of the requested steps as fit REF_BUDGET_S
    tw = time.perf_counter()
    warm = 0
    for _ in range(args.warmup):
        run()
        warm += 1
        if time.perf_counter() - tw > REF_BUDGET_S / 6:
            break
    per = (time.perf_counter() - tw) / max(warm, 1)
    steps = max(1, min(args.steps, int(REF_BUDGET_S // max(per, 1e-9))))
    el = sum(run() for _ in range(steps))
    value = steps * units / el
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
        "steps": steps, "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 * el / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "d": dims[0], "hidden": dims[1], "layers": dims[2]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": T, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_apply(cfg_name, seconds=20.0):
    """Our line's cpu_baseline: the reference apply, ONE thread (the reference
    apply is single-threaded, src/gnn.cpp:120-206), bounded sample."""
    run, units, desc, kind, T = ref_apply_sampler(cfg_name, threads=1)
    reps, total = 0, 0.0
    while total < seconds and reps < 50:
        total += run()
        reps += 1
    return {"value": reps * units / total, "unit": "applies/s", "cores": 1, "kind": kind,
            "sample": f"{reps} step(s) of: {desc}; {total:.1f} s"}


def cpu_baseline_train():
    run, units, desc, kind, T = ref_train_sampler()
    el = run()
    return {"value": units / el, "unit": "steps/s", "cores": T, "kind": kind,
            "sample": f"1 step of: {desc}; {el:.1f} s (a C3 step extrapolated from it)"}


# --------------------------------------------------------------- our arm
def build_workload(capi, cfg_name):
    cfg = CONFIGS[cfg_name]
    kind, size, p0, p1, seed = cfg["gen"]
    a = capi.Csr.generate(kind, size, p0, p1, seed)
    ah = a.prescale(a.gamma())
    n, nnz = ah.info()
    params = capi.init_params(*cfg["dims"], 0)
    model = capi.Model(ah, cfg["dims"], params)
    rk, rs = cfg["rhs"]
    b = capi.gaussian_vector(rs, n) if rk == "gauss" else ah.spmv(capi.gaussian_vector(rs, n))
    return dict(name=cfg_name, cfg=cfg, a=ah, n=n, nnz=nnz, dims=cfg["dims"], params=params,
                model=model, b=b)


def apply_leg(capi, torch, cfg_name, args, rank, world, dist, local, full=True):
    """Apply throughput (device-resident), roofline of the dominant kernel,
    e2e through gnpc_apply with host buffers, one FGMRES solve."""
    w = build_workload(capi, cfg_name)
    n, nnz, (d, hdim, L) = w["n"], w["nnz"], w["dims"]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    model = w["model"]
    nb = 8  # distinct right-hand sides resident in HBM
    rng = np.random.default_rng(1234 + rank)
    bs = [torch.tensor(w["b"] * (1.0 + 0.01 * rng.standard_normal()), dtype=torch.float32, device="cuda")
          for _ in range(nb)]
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def do_step(i):
        model.apply_device_f32(bs[i % nb].data_ptr(), out.data_ptr(), sptr)

    clocks = ClockSampler(local)
    clocks.start()
    for i in range(args.warmup):
        flush.zero_()
        do_step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = capi.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        do_step(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    launches = capi.launch_count() - l0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = sum(s.elapsed_time(e) for s, e in evs)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * args.steps / (max_ms / 1e3)
    step_ms = max_ms / args.steps

    # ---- roofline: per-kernel CUDA events on the launching stream
    dp = dp_of(d)
    sell, longr = w["a"].device_layout()[1:3]
    lflags = w["a"].layout_flags()
    if dp == 32 and lflags & 4:
        layer_kernel = ("k_layer_sell<DP=32, strip windows> (fused Res-GCONV: X row windows staged in shared "
                        "memory by TMA along strips of the dominant tile stride, pair-union entries, tcgen05 "
                        "3xTF32; MMA warp + TMA producer warp)")
    elif dp == 32 and lflags & 2:
        layer_kernel = "k_layer_sell<DP=32, pair-union> (fused Res-GCONV, pair-union sliced-ELL TMA pipeline, tcgen05 3xTF32)"
    elif dp in (16, 32) and sell:
        layer_kernel = f"k_layer_sell<DP={dp}> (fused Res-GCONV, sliced-ELL TMA pipeline, tcgen05 3xTF32)"
    elif dp in (16, 32):
        layer_kernel = (f"k_layer_sell<DP={dp}, CSR> (fused Res-GCONV, short-row CSR TMA pipeline, "
                        "tcgen05 3xTF32)" + (" + long-row chunks" if longr else ""))
    else:
        layer_kernel = f"k_layer<DP={dp}> (fused Res-GCONV, CUDA cores)"
    ms_k = np.zeros(5)
    cnt_k = np.zeros(5, np.int64)
    for i in range(args.steps):
        flush.zero_()
        model.apply_profile(bs[i % nb].data_ptr(), out.data_ptr(), sptr, ms_k, cnt_k)
    # d = 32 strip windows: the lift is fused into the first layer's kernel
    # (k_layer_sell_lift), which gnpc_apply_profile times in the lift's slot
    lift_fused = bool(dp == 32 and lflags & 4 and cnt_k[3] == (L - 2) * args.steps and cnt_k[1] == args.steps)
    mid_ms = ms_k[3] / max(1, cnt_k[3])
    long_ms = ms_k[2] / max(1, cnt_k[2]) if cnt_k[2] else 0.0
    peak, peak_src = load_peaks()
    lb = layer_bytes(n, nnz, dp)
    # a layer over a matrix with long rows is two launches (chunks + fused
    # layer): its time is their sum
    layer_ms = mid_ms + (long_ms * cnt_k[2] / max(1, cnt_k[3] + cnt_k[4]) if cnt_k[2] else 0.0)
    achieved = lb / (layer_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg_name}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    ab = apply_bytes(n, nnz, dp, L)
    apply_gbs = ab / (step_ms / 1e3) / 1e9
    per_layer = {"kernel": layer_kernel, "algorithmic_bytes_per_launch": lb, "avg_launch_ms": layer_ms,
                 "achieved_gbs": achieved, "frac": achieved / peak,
                 "timing": "separate per-layer launches, CUDA events per kernel (gnpc_apply_profile)"}
    if launches == args.steps:
        # one launch per apply: the persistent whole-apply kernel is the only
        # kernel; its bytes are the apply's canonical bytes
        roof = {"bound": "hbm", "achieved": apply_gbs, "peak": peak, "unit": "GB/s",
                "frac": apply_gbs / peak, "traffic": traffic,
                "kernel": f"k_apply_sell<DP={dp}> (whole apply in one persistent cooperative launch)",
                "algorithmic_bytes_per_launch": ab, "avg_launch_ms": step_ms, "peak_source": peak_src,
                "kernel_share_of_step": 1.0, "per_layer_launches": per_layer}
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": layer_kernel,
                "algorithmic_bytes_per_launch": lb, "avg_launch_ms": layer_ms, "peak_source": peak_src,
                "kernel_share_of_step": float((ms_k[2] + ms_k[3] + ms_k[4] + (ms_k[1] if lift_fused else 0.0))
                                              / max(ms_k.sum(), 1e-12)),
                "timing": "CUDA events around every launch on the launching stream (gnpc_apply_profile)"}
        if lift_fused:
            roof["note"] = ("avg_launch_ms is the plain layer kernel (layers 2..L-1); the first layer runs "
                            "k_layer_sell_lift (lift fused: its row windows are computed in shared memory, x1 "
                            "never crosses HBM), timed under per_kernel_ms.lift_and_first_layer")

    # ---- e2e through the C ABI with pinned host f64 buffers
    import ctypes as C

    hb = torch.tensor(w["b"], dtype=torch.float64).pin_memory()
    ho = torch.empty(n, dtype=torch.float64).pin_memory()
    lib = capi.lib()
    for _ in range(3):
        capi.check(lib.gnpc_apply(model.h, C.c_void_p(hb.data_ptr()), C.c_void_p(ho.data_ptr())))
    e2e_steps = args.steps
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        capi.check(lib.gnpc_apply(model.h, C.c_void_p(hb.data_ptr()), C.c_void_p(ho.data_ptr())))
    e2e_el = time.perf_counter() - t0
    te = torch.tensor([e2e_el], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": world * e2e_steps / float(te.item()), "unit": "applies/s",
           "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
           "api": "gnpc_apply (host f64, pinned)"}

    # ---- one FGMRES solve (device-resident), with its byte model
    fg = None
    if not args.no_fgmres:
        restart, rtol, maxiters = w["cfg"]["fg"]
        bd = torch.tensor(w["b"], dtype=torch.float64, device="cuda")
        xd = torch.zeros(n, dtype=torch.float64, device="cuda")
        capi.fgmres_device(w["a"], model, bd.data_ptr(), xd.data_ptr(), rtol, 2, restart, sptr)
        xd.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = capi.fgmres_device(w["a"], model, bd.data_ptr(), xd.data_ptr(), rtol, maxiters, restart, sptr)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        its = s["history"][-1][0]
        fb = fgmres_bytes(n, nnz, dp, L, its, restart, s["reorth_steps"])
        fg = {"solve_s": el, "iterations": its, "status": s["status"],
              "final_relres": s["history"][-1][1], "restart": restart, "rtol": rtol,
              "maxiters": maxiters, "reorth_steps": s["reorth_steps"],
              "ms_per_iteration": 1e3 * el / max(1, its),
              "krylov_ms_per_iteration": 1e3 * el / max(1, its) - step_ms,
              "algorithmic_bytes": fb, "achieved_gbs": fb / el / 1e9, "frac": fb / el / 1e9 / peak,
              "bytes_model": "SURVEY §8d per-iteration model (apply + SpMV + MGS 40n(j+1) per pass "
                             "+ norms/normalise/z; per cycle x += Zy and true residual); re-orth passes "
                             "counted exactly, charged at the solve's mean basis length",
              "timing": "host wall clock around gnpc_fgmres_device with device syncs on both sides"}
    leg = {
        "value": value, "unit": "applies/s", "ms_per_step": step_ms, "steps": args.steps,
        "config": {"workload": w["cfg"]["desc"], "n": n, "nnz": nnz, "d": d, "hidden": hdim, "layers": L,
                   "rhs": "8 distinct resident RHS, fp32",
                   "l2": "flushed between timed steps (512 MiB write, untimed)",
                   "parallelism": f"replicas x{world}"},
        "roofline": roof, "apply_gbs": apply_gbs, "apply_frac_of_peak": apply_gbs / peak,
        "e2e": e2e, "clocks": clk, "gpu_launches": int(launches), "fgmres": fg,
        "per_kernel_ms": {"norm": ms_k[0] / max(1, cnt_k[0]),
                          ("lift_and_first_layer" if lift_fused else "lift"): ms_k[1] / max(1, cnt_k[1]),
                          "long_rows": long_ms if cnt_k[2] else None, "layer": mid_ms,
                          "last_layer_projection": ms_k[4] / max(1, cnt_k[4])},
    }
    del bs, out, flush
    return leg


def train_leg(capi, torch, args, rank, world, dist, local):
    """C3: batched GNP training, 2D var-coeff diffusion 512^2, d=32, B=32.

    value: the reference's train_preconditioner step (src/gnn.cpp:416-449):
    pairs x ~ N(0,I) from the reference Rng stream (mt19937_64 words from a
    host thread, Box-Muller and b = A x on the device), forward, L1 loss,
    backward, Adam, then the monitoring forward on the fixed 16-column batch
    and the best snapshot, all device-resident (gnpc_train_run).  The pure
    training step (device Philox pairs, no monitor), the monitoring forward and
    the pair generation are also timed on their own."""
    kind, size, p0, p1, seed = C3["gen"]
    B, MB = C3["batch"], C3["monitor"]
    a = capi.Csr.generate(kind, size, p0, p1, seed)
    ah = a.prescale(a.gamma())
    n, nnz = ah.info()
    dims = C3["dims"]
    m = capi.Model(ah, dims, capi.init_params(*dims, 0))
    t = capi.Trainer(m, B, lr=1e-3)
    ts = torch.cuda.ExternalStream(t.stream())
    if dist:
        from paper_2406_00809_b200.dp import DataParallelTrainer, TrainerEngine

        dp = DataParallelTrainer(TrainerEngine(t))
        do = dp.step_synthetic
    else:
        do = t.step_synthetic
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        do(1000)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    l0 = capi.launch_count()
    # events on the trainer's own (non-blocking) stream, which every kernel of
    # the step runs on
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ts)
    losses = [do(1000) for _ in range(args.steps)]
    ev1.record(ts)
    torch.cuda.synchronize()
    launches = capi.launch_count() - l0
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    max_ms = float(tt.item())
    peak, peak_src = load_peaks()
    sb = train_step_bytes(n, nnz, dims[0], B, dims[2])
    step_ms = max_ms / args.steps
    leg = {
        "value": world * args.steps / (max_ms / 1e3), "unit": "steps/s", "ms_per_step": step_ms,
        "steps": args.steps,
        "config": {"workload": C3["desc"], "n": n, "nnz": nnz, "batch": B, "global_batch": B * world,
                   "parallelism": f"dp{world} (gradient all-reduce, NCCL)" if world > 1 else "dp1",
                   "l2": "activations 18 GiB >> L2 (no flush needed)",
                   "step": "device Philox pairs (x ~ N(0,I), b = A x), forward, L1 loss, backward, Adam"},
        "roofline": {"bound": "hbm", "achieved": sb / (step_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": sb / (step_ms / 1e3) / 1e9 / peak, "traffic": None,
                     "algorithmic_bytes_per_step": sb, "peak_source": peak_src, "kernel": "whole training step"},
        "loss_first_last": [losses[0], losses[-1]], "clocks": clk, "gpu_launches": int(launches),
    }
    if world == 1:
        leg["train_preconditioner"] = train_run_leg(capi, torch, ah, n, nnz, dims, B, MB, args, peak)
        leg["e2e"] = train_e2e(capi, torch, t, ah, n, B, ts, args)
    return leg


def train_run_leg(capi, torch, ah, n, nnz, dims, B, MB, args, peak):
    """The reference-API training loop on the device (gnpc_train_run): per
    step, reference-stream Gaussian pairs (host mt19937_64 words, device
    Box-Muller, device b = A x in f64), forward/loss/backward/Adam, monitor
    forward and best snapshot; losses stay on the device until the end."""
    if not hasattr(capi, "train_run"):
        return None
    steps = max(args.steps, 20)
    r = capi.train_run(ah, dims=dims, steps=steps, batch=B, spectral=0, arnoldi_m=10, seed=0,
                       monitor_batch=MB, timing=True)
    tm = r["timing"]
    out = {"steps": steps, "ms_per_step": tm["ms_per_step"], "steps_per_s": 1e3 / tm["ms_per_step"],
           "monitor_ms_per_step": tm["monitor_ms"], "pairgen_ms_per_step": tm["pairgen_ms"],
           "monitor_gbs": monitor_bytes(n, nnz, dims[0], MB, dims[2]) / (tm["monitor_ms"] / 1e3) / 1e9
           if tm["monitor_ms"] > 0 else None,
           "pairgen_gbs": pair_bytes(n, nnz, B) / (tm["pairgen_ms"] / 1e3) / 1e9 if tm["pairgen_ms"] > 0 else None,
           "loss_first_last": [float(r["losses"][0]), float(r["losses"][-1])], "best_loss": r["best_loss"],
           "timing": tm.get("how")}
    return out


def train_e2e(capi, torch, t, ah, n, B, ts, args):
    """gnpc_train_step with pinned host n x B f64 x and b copied in every step
    and the loss read back."""
    xh = torch.empty((B, n), dtype=torch.float64, pin_memory=True).numpy()
    bh = torch.empty((B, n), dtype=torch.float64, pin_memory=True).numpy()
    rng = np.random.default_rng(5)
    xh[:] = rng.standard_normal((B, n))
    for k in range(B):
        bh[k] = ah.spmv(xh[k])
    xf, bf = xh.reshape(-1), bh.reshape(-1)
    for _ in range(2):
        t.step(xf, bf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne = max(3, min(args.steps, 10))
    e0.record(ts)
    for _ in range(ne):
        t.step(xf, bf)
    e1.record(ts)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / ne
    return {"value": 1e3 / ems, "unit": "steps/s", "h2d_bytes_per_step": 2 * 8 * n * B,
            "d2h_bytes_per_step": 8, "api": "gnpc_train_step (host f64 x, b; pinned)"}


def summarize(leg):
    keep = ("value", "unit", "ms_per_step", "config", "roofline", "apply_gbs", "apply_frac_of_peak", "e2e",
            "fgmres", "per_kernel_ms", "gpu_launches", "clocks", "train_preconditioner", "loss_first_last")
    return {k: leg[k] for k in keep if k in leg}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS) + ["c3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fgmres", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline config only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    default_run = "--config" not in " ".join(sys.argv)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2406_00809_b200 import capi

    capi.check(capi.lib().gnpc_set_device(local))
    if args.config == "c3":
        leg = train_leg(capi, torch, args, rank, world, dist, local)
        metric = C3_METRIC
    else:
        leg = apply_leg(capi, torch, args.config, args, rank, world, dist, local)
        metric = METRIC
    extras = {}
    if default_run and not args.no_extras and world == 1:
        # the other north-star configs, same run (informational; each carries
        # its own roofline / FGMRES / e2e)
        for c in ("c4", "c2"):
            extras[c] = summarize(apply_leg(capi, torch, c, args, rank, world, dist, local))
        extras["c3"] = summarize(train_leg(capi, torch, args, rank, world, dist, local))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_train() if args.config == "c3" else cpu_baseline_apply(args.config)
    if rank == 0:
        line = {"metric": metric, "value": leg["value"], "unit": leg["unit"], "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": leg["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic", "config": leg["config"], "roofline": leg["roofline"],
                "cpu_baseline": cpu, "e2e": leg.get("e2e"), "clocks": leg["clocks"],
                "gpu_launches": leg["gpu_launches"]}
        for k in ("apply_gbs", "apply_frac_of_peak", "fgmres", "per_kernel_ms", "train_preconditioner",
                  "loss_first_last"):
            if k in leg:
                line[k] = leg[k]
        if extras:
            line["configs"] = extras
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
