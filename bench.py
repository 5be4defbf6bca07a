"""Benchmark driver (contract: see DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json `metric`: "fp64 TFLOP/s precond+GENP at n=8192; batched n=64
solves/s; % of roofline"):
  * headline `value` — config 3: Gaussian-preconditioned GENP, n = 8192, 16 RHS, MulSide::Right
    (G = gaussian_matrix(n, n) on the reference's Right stream, A G, blocked GENP with block 128,
    forward/back solves, X = G Y, residual-gated acceptance).  TFLOP/s over the algorithmic
    1.4704e12 flop of SURVEY.md §8(d) (A G + LU + solves + G Y; G generation is timed but not
    counted).  Inputs resident in HBM; A (512 MiB) and G (512 MiB) exceed the 126 MB L2.
  * `batched` — config 2: 4096 systems of n = 64 with circulant +-1 multipliers (solves/s).
  * `config1` — n = 256 (latency): us per solve on device data and through the host-pointer call.
  * `config5` — n = 16384, 8 RHS, with the Householder-pair, sparse +-1 and Gaussian right
    multipliers (ms per call, attempts, backward error; 1 warm-up + 2 timed calls per arm;
    `--skip-config5` leaves it out); the structured arms add `multiplier_apply`, the matrix-free
    multiplier stage alone with its HBM fraction.
  * `circulant_fft` — A C for a circulant +-1 right multiplier at n = 8192 through the FFT path,
    beside the dense DMMA product it replaces.
  * `range_finder` — config 4: the randomized range finder on A 16384 x 4096, rho+ = 72
    (TFLOP/s over SURVEY.md §8(d)'s 1.967e10 flop); for N > 1 the rows are sharded (TSQR of
    the sketch + one all_reduce of B, strong scaling).
  * `e2e` — the same config-3 solve through the public host-pointer C-ABI call
    (rl_randomized_genp_ex) from pinned host buffers: H2D of A and B, D2H of X inside the timed
    region.
One process per GPU; for N > 1 (torchrun) every rank runs an independent replica of the
config-3 solve (the path does not shard: "replicas only") and its own 4096-system
batch (weak scaling); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 TFLOP/s precond+GENP at n=8192; batched n=64 solves/s; % of roofline"
N3, NRHS3 = 8192, 16
FLOPS3 = 2 * N3 ** 3 + 2 * N3 ** 3 / 3 + 2 * N3 ** 2 * NRHS3 + 2 * N3 ** 2 * NRHS3   # 1.4704e12
N1 = 256
FLOPS1 = 2 * N1 ** 3 + 2 * N1 ** 3 / 3 + 2 * N1 ** 2 + 2 * N1 ** 2   # 45.00 MFLOP
N5, NRHS5 = 16384, 8
FLOPS5_G = 2 * N5 ** 3 + 2 * N5 ** 3 / 3 + 2 * N5 ** 2 * NRHS5 * 2   # C5 Gaussian arm per attempt
FLOPS5_LU = 2 * N5 ** 3 / 3
M4, N4, R4, K4 = 16384, 4096, 64, 72
FLOPS4 = 2 * M4 * N4 * K4 * 2 + 3.4e8   # Y = A H + QR(Y) + B = Q^T A: 1.967e10
BATCH2, N2 = 4096, 64
FLOPS2_PER_SYS = 445035      # circulant signed sums + LU + solves + C y
BYTES2_PER_SYS = 33800
SEED = 20260825


# ----------------------------------------------------------------- helpers ----
def shard_range(total: int, rank: int, world: int):
    """Contiguous block of [0, total) owned by `rank` (independent units, no collective)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    In-process NVML (pynvml) every 200 ms when available — a spawned `nvidia-smi -lms 100`
    measurably perturbs the timed region (tools/c3_overhead.py: +7% on config 3) — else the
    nvidia-smi query loop.  Rows: sm, max sm, active, hw_slowdown, hw_thermal, sw_thermal,
    sw_power_cap."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0, period_s: float = 0.2):
        self.index = index
        self.period = period_s
        self.rows = []
        self.proc = None
        self.thread = None
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), hex(rs)] + ["Active" if rs & b else "Not Active" for b in bits])
            except Exception:  # noqa: BLE001
                break
            self.stop.wait(self.period)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.nvml:
            self.stop.set()
            self.thread.join(timeout=5)
            return False
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def config3(world):
    """The headline workload (BASELINE.json configs[2]); identical in both arms' JSON lines."""
    return {"workload": "config3: Gaussian-preconditioned GENP n=8192, 16 RHS, MulSide::Right, block 128",
            "n": N3, "nrhs": NRHS3, "flop_per_attempt": FLOPS3, "parallelism": f"replicas{world}",
            "l2": "inputs larger than L2 (A, G 512 MiB each)"}


def make_config3_inputs(torch, dev):
    """A = U diag(sigma) V^T-like test matrix of config 3, built once on the GPU (not timed).

    Construction: A = Q1 diag(sigma) Q2^T with Q1, Q2 the Q
    factors of seeded Gaussians (torch's QR on device, input construction only), sigma log-spaced
    1 .. 1e-6, then the leading 4096^2 block replaced by P Q (4096 x 4095 times 4095 x 4096), with
    the Gaussians drawn from the reference's own streams by the library (bit-exact draws).
    """
    import paper_1212_4560_b200 as rl
    n, h = N3, N3 // 2
    g1 = torch.empty(n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(g1, 0.0, 1.0, rl.RngStream(SEED, 31))
    q1, _ = torch.linalg.qr(g1)
    rl.dev_gaussian_matrix(g1, 0.0, 1.0, rl.RngStream(SEED, 32))
    q2, _ = torch.linalg.qr(g1)
    sig = torch.logspace(0, -6, n, dtype=torch.float64, device=dev)
    A = (q1 * sig) @ q2.T
    del q1, q2
    P = torch.empty(h, h - 1, dtype=torch.float64, device=dev)
    Q = torch.empty(h - 1, h, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(P, 0.0, 1.0, rl.RngStream(SEED, 33))
    rl.dev_gaussian_matrix(Q, 0.0, 1.0, rl.RngStream(SEED, 34))
    A[:h, :h] = P @ Q
    Xt = torch.empty(n, NRHS3, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(Xt, 0.0, 1.0, rl.RngStream(SEED, 35))
    B = A @ Xt
    del g1, P, Q
    torch.cuda.synchronize()
    return A.contiguous(), B.contiguous()


def make_config2_inputs(torch, dev, batch):
    import paper_1212_4560_b200 as rl
    n = N2
    A = torch.empty(batch, n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(A.view(batch * n, n), 0.0, 1.0, rl.RngStream(SEED, 41))
    P = torch.empty(batch, 32, 31, dtype=torch.float64, device=dev)
    Q = torch.empty(batch, 31, 32, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(P.view(batch * 32, 31), 0.0, 1.0, rl.RngStream(SEED, 42))
    rl.dev_gaussian_matrix(Q.view(batch * 31, 32), 0.0, 1.0, rl.RngStream(SEED, 43))
    A[:, :32, :32] = torch.bmm(P, Q)
    xt = torch.empty(batch, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(xt, 0.0, 1.0, rl.RngStream(SEED, 44))
    b = torch.bmm(A, xt.unsqueeze(2)).squeeze(2).contiguous()
    sids = torch.arange(batch, dtype=torch.int64, device=dev) + 7
    torch.cuda.synchronize()
    return A.contiguous(), b, sids


def _timed(torch, fn, warmup, steps, dist):
    for _ in range(warmup):
        out = fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return max_over_ranks(e0.elapsed_time(e1) / steps, dist), out


def run_config1(torch, rl, dev, dist, args, fp64_peak):
    """Config 1: n = 256 Gaussian-preconditioned GENP, MulSide::Right, one RHS (latency-bound):
    A with its leading 128^2 block = P Q (rank 127), x_true, b = A x_true."""
    n, h = N1, N1 // 2
    A = torch.empty(n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(SEED, 11))
    P = torch.empty(h, h - 1, dtype=torch.float64, device=dev)
    Q = torch.empty(h - 1, h, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(P, 0.0, 1.0, rl.RngStream(SEED, 12))
    rl.dev_gaussian_matrix(Q, 0.0, 1.0, rl.RngStream(SEED, 13))
    A[:h, :h] = P @ Q
    xt = torch.empty(n, 1, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(xt, 0.0, 1.0, rl.RngStream(SEED, 14))
    b = (A @ xt).contiguous()
    x = torch.empty_like(b)
    kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
    st = rl.RngStream(SEED, 15)
    ms, rep = _timed(torch, lambda: rl.dev_randomized_genp(A, b, x, kind, rl.MulSide.RIGHT, 0, st,
                                                           skip_raw_arm=True),
                     max(args.warmup, 3), max(args.steps, 20), dist)
    bwd = float(((A @ x - b).norm() / (A.norm() * x.norm())).item())
    # the same solve from host buffers through the public host-pointer call
    hA, hb, hx = A.cpu().numpy(), b.cpu().numpy().ravel(), np.empty(n)
    for _ in range(max(args.warmup, 3)):  # the host path's own warm-up (its contrast-arm helper thread)
        rl.randomized_genp(hA, hb, kind, rl.MulSide.RIGHT, 0, st)
    t0 = time.perf_counter()
    reps = max(args.steps, 20)
    for _ in range(reps):
        rl.randomized_genp(hA, hb, kind, rl.MulSide.RIGHT, 0, st)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / reps, dist)
    cpu1 = cpu_baseline_config1(hA, hb) if (not dist and not args.no_cpu_baseline) else None
    return {"workload": "config1: Gaussian-preconditioned GENP n=256, 1 RHS, MulSide::Right (latency)",
            "cpu_baseline": cpu1,
            "value_us_per_solve": round(ms * 1e3, 2), "attempts": rep.attempts_drawn,
            "tflops_executed": round(rep.attempts_drawn * FLOPS1 / (ms * 1e-3) / 1e12, 5),
            "flop_per_attempt": FLOPS1, "backward_error": bwd, "residual": rep.residual,
            "e2e_us_per_solve": round(e2e_ms * 1e3, 1),
            "e2e_call": "rl_randomized_genp (host pointers, contrast arm included, as the reference)",
            "roofline": {"bound": "latency", "frac_fp64": round(FLOPS1 / (ms * 1e-3) / 1e12 / fp64_peak, 6)}}


def make_config5_inputs(torch, dev):
    """Config 5: A 16384^2 Gaussian with its leading 8192^2 block = P Q (rank 8191), X_true
    16384 x 8, B = A X_true; built once on the GPU, not timed."""
    import paper_1212_4560_b200 as rl
    n, h = N5, N5 // 2
    A = torch.empty(n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(SEED, 51))
    P = torch.empty(h, h - 1, dtype=torch.float64, device=dev)
    Q = torch.empty(h - 1, h, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(P, 0.0, 1.0, rl.RngStream(SEED, 52))
    rl.dev_gaussian_matrix(Q, 0.0, 1.0, rl.RngStream(SEED, 53))
    A[:h, :h] = P @ Q
    del P, Q
    Xt = torch.empty(n, NRHS5, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(Xt, 0.0, 1.0, rl.RngStream(SEED, 54))
    B = (A @ Xt).contiguous()
    torch.cuda.synchronize()
    return A, B


def hbm_reference_peak(hbm_same_run):
    """HBM roofline denominator: MEASURED_PEAKS.json's driver-measured copy bandwidth when the
    file is present, else this run's own copy probe."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy)"
    except (OSError, KeyError, ValueError):
        return hbm_same_run, "same-run copy probe (rl_probe_peaks)"


def time_multiplier_apply(torch, rl, dev, dist, tag, A, mult_bytes, hbm_peak):
    """The structured multiplier stage alone (the HBM-bound kernels of config 5): A S with its
    gather plan (k_sparse_plan + k_sparse_right4), or A H1 H2 (k_dot_pm1 + k_hh2_onepass: A read once),
    at n = 16384 through the device C-ABI; A (2 GiB) and the output exceed L2, so no flush
    is needed between calls.  Algorithmic bytes: 2 n^2 8 for both (A read once, A M written once)."""
    n = A.shape[0]
    out = torch.empty_like(A)
    if tag == rl.MultiplierTag.SPARSE_SIGN:
        rows_h, signs_h = rl.sparse_sign(n, rl.RngStream(SEED, 56))
        rows, signs = torch.from_numpy(rows_h).to(dev), torch.from_numpy(signs_h).to(dev)
        fn = lambda: rl.dev_sparse_apply_right(rows, signs, A, out)  # noqa: E731
        kernels = "k_sparse_plan + k_sparse_right4"
    else:
        u = torch.from_numpy(rl.rng_draws(rl.RngStream(SEED, 57), "sign", 2 * n)).to(dev)
        u1, u2 = u[:n].contiguous(), u[n:].contiguous()
        fn = lambda: rl.dev_householder_pair_apply_right(u1, u2, A, out)  # noqa: E731
        kernels = "k_dot_pm1 + k_hh2_onepass"
    ms, _ = _timed(torch, fn, 3, 20, dist)
    peak, src = hbm_reference_peak(hbm_peak)
    gbs = mult_bytes / (ms * 1e-3) / 1e9
    del out
    return {"kernels": kernels, "ms": round(ms, 4), "achieved_gbs": round(gbs, 1), "peak_gbs": peak,
            "frac": round(gbs / peak, 4), "peak_source": src, "frac_same_run_copy": round(gbs / hbm_peak, 4)}


def run_circulant_fft(torch, rl, dev, dist, hbm_peak):
    """a circulant +-1 right multiplier at n = 8192 applied matrix-free
    (randomized_genp's Right-side A C through k_circ_fft_prep + k_circ_right_fft) against the
    dense DMMA product it replaces; HBM roofline over 2 n^2 8 bytes (A read once, A C written
    once; A and A C exceed L2)."""
    n = 8192
    A = torch.empty(n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(SEED, 71))
    c = torch.from_numpy(rl.rng_draws(rl.RngStream(SEED, 72), "sign", n)).to(dev)
    out = torch.empty_like(A)
    ms, _ = _timed(torch, lambda: rl.dev_circulant_apply_right(c, A, out), 3, 20, dist)
    idx = (torch.arange(n, device=dev)[:, None] - torch.arange(n, device=dev)[None, :]) % n
    C = c[idx]
    ref = torch.empty_like(A)
    ms_dense, _ = _timed(torch, lambda: rl.dev_gemm(A, C, ref), 1, 2, dist)
    diff = float((out - ref).abs().max() / ref.abs().max())
    peak, src = hbm_reference_peak(hbm_peak)
    gbs = 2.0 * n * n * 8 / (ms * 1e-3) / 1e9
    del A, out, C, ref
    torch.cuda.empty_cache()
    return {"workload": "A C, circulant +-1 right multiplier, n = 8192 (FFT path)", "ms": round(ms, 4),
            "dense_dmma_ms": round(ms_dense, 3), "max_rel_diff_vs_dense": diff,
            "roofline": {"bound": "hbm", "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 4),
                         "peak_source": src}}


def run_config5(torch, rl, dev, dist, args, fp64_peak, hbm_peak, rank=0, world=1):
    """Config 5: n = 16384, 8 RHS, MulSide::Right with the orthogonal Householder pair, the
    sparse +-1 and the Gaussian multipliers (contrast arm skipped as in config 3).  Short runs
    (1 warm-up + 2 timed calls per arm: a Gaussian call is ~1 s)."""
    A, B = make_config5_inputs(torch, dev)
    X = torch.empty_like(B)
    out = {"workload": "config5: GENP n=16384, 8 RHS, MulSide::Right; Householder pair / sparse +-1 / Gaussian"}
    arms = (("householder_pair", rl.MultiplierTag.HOUSEHOLDER_PAIR, 2.0 * N5 * N5 * 8),
            ("sparse_sign", rl.MultiplierTag.SPARSE_SIGN, 2.0 * N5 * N5 * 8),
            ("gaussian", rl.MultiplierTag.GAUSSIAN, None))
    for name, tag, mult_bytes in arms:
        kind = rl.MultiplierKind(tag)
        st = rl.RngStream(SEED, 55)
        ms, rep = _timed(torch, lambda: rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, st,
                                                               skip_raw_arm=True), 1, 2, dist)
        bwd = float(((A @ X - B).norm(dim=0) / (A.norm() * X.norm(dim=0))).max().item())
        arm = {"ms_per_call": round(ms, 2), "attempts": rep.attempts_drawn, "residual": rep.residual,
               "backward_error_max": bwd}
        if tag == rl.MultiplierTag.GAUSSIAN:
            arm["tflops_executed"] = round(rep.attempts_drawn * FLOPS5_G / (ms * 1e-3) / 1e12, 3)
            arm["frac_fp64"] = round(arm["tflops_executed"] / fp64_peak, 4)
        else:
            arm["lu_tflops_executed"] = round(rep.attempts_drawn * FLOPS5_LU / (ms * 1e-3) / 1e12, 3)
            arm["multiplier_bytes_per_apply"] = mult_bytes
            arm["multiplier_apply"] = time_multiplier_apply(torch, rl, dev, dist, tag, A, mult_bytes, hbm_peak)
        out[name] = arm
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline_config5(A.cpu().numpy(), os.cpu_count() or 1)
        for name in ("householder_pair", "sparse_sign", "gaussian"):
            out[name]["cpu_baseline"] = cb[name]
    del A, B, X
    torch.cuda.empty_cache()
    return out


def make_config4_rows(torch, dev, lo, hi):
    """Rows [lo, hi) of the config-4 matrix A = U diag(logspace(0,-2,64)) V^T + 1e-10 E
    (SURVEY.md §8(d)); U, V are the Q factors of seeded Gaussians (input construction, not
    the measured path), identical on every rank."""
    import paper_1212_4560_b200 as rl
    g1 = torch.empty(M4, R4, dtype=torch.float64, device=dev)
    g2 = torch.empty(N4, R4, dtype=torch.float64, device=dev)
    E = torch.empty(M4, N4, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(g1, 0.0, 1.0, rl.RngStream(SEED, 61))
    rl.dev_gaussian_matrix(g2, 0.0, 1.0, rl.RngStream(SEED, 62))
    rl.dev_gaussian_matrix(E, 0.0, 1.0, rl.RngStream(SEED, 63))
    U, _ = torch.linalg.qr(g1)
    V, _ = torch.linalg.qr(g2)
    sig = torch.logspace(0, -2, R4, dtype=torch.float64, device=dev)
    A = ((U[lo:hi] * sig) @ V.T + 1e-10 * E[lo:hi]).contiguous()
    del E, g1, g2
    torch.cuda.synchronize()
    return A


def run_config4(torch, rl, dev, dist, rank, world, args, fp64_peak):
    """Config 4: the randomized range finder, 16384 x 4096, rho+ = 72, rank tol 1e-8.  N = 1:
    the fused device path (rl_dev_range_finder).  N > 1: rows sharded across ranks (strong
    scaling), TSQR + one all_reduce (paper_1212_4560_b200/sharded.py); time = max over ranks."""
    from paper_1212_4560_b200.sharded import DistGroup, range_finder_sharded
    lo, hi = shard_range(M4, rank, world)
    A = make_config4_rows(torch, dev, lo, hi)
    st = rl.RngStream(SEED, 64)
    Q = torch.empty(hi - lo, K4, dtype=torch.float64, device=dev)
    B = torch.empty(K4, N4, dtype=torch.float64, device=dev)
    group = DistGroup(dist) if dist else None
    resid = None
    if world == 1:
        _, rk, resid = rl.dev_range_finder(A, K4, st, 1e-8, Q, B, want_residual=True)

        def step():
            return rl.dev_range_finder(A, K4, st, 1e-8, Q, B, want_residual=False)[1]
    else:
        def step():
            return range_finder_sharded(A, K4, st, 1e-8, group)[1]
        rk = step()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    k4 = max(args.steps, 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k4):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms4 = max_over_ranks(e0.elapsed_time(e1) / k4, dist)
    tf4 = FLOPS4 / (ms4 * 1e-3) / 1e12
    cpu4 = None
    if world == 1 and not args.no_cpu_baseline:
        H = torch.empty(N4, K4, dtype=torch.float64, device=dev)
        rl.dev_gaussian_matrix(H, 0.0, 1.0, st)
        cpu4 = cpu_baseline_config4(A[:2048].cpu().numpy(), H.cpu().numpy())
    del A, Q, B
    out = {"workload": "config4: range finder Y = A H, qr_positive(Y), B = Q^T A, numerical_rank(B, 1e-8); "
                       "A 16384 x 4096, rho+ = 72",
           "value": round(tf4, 4), "unit": "TFLOP/s", "ms_per_step": round(ms4, 4), "flop": FLOPS4,
           "rank": rk, "parallelism": "fused" if world == 1 else f"rows{world} (TSQR + all_reduce of B)",
           "scaling": "strong",
           "roofline": {"bound": "fp64", "frac": round(tf4 / fp64_peak, 4), "peak": round(fp64_peak, 3),
                        "roofline_ms": round(FLOPS4 / (fp64_peak * 1e12) * 1e3, 4)}}
    if resid is not None:
        out["resid_fro"] = resid
    if cpu4 is not None:
        out["cpu_baseline"] = cpu4
    return out


def load_profile_traffic():
    """Per-launch DRAM traffic of the dominant kernel from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------ our arm ----
def run_ours(args, dist, rank, world, local_rank):
    import torch
    import paper_1212_4560_b200 as rl
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    rl.lib().rl_init(local_rank)
    fp64_peak, hbm_peak = rl.probe_peaks()

    kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
    A, B = make_config3_inputs(torch, dev)
    X = torch.empty_like(B)
    stream = rl.RngStream(SEED, 11)

    def step3():
        return rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, stream, skip_raw_arm=True)

    for _ in range(args.warmup):
        rep = step3()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rl.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            rep = step3()
        e1.record()
        torch.cuda.synchronize()
    launches = rl.launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        dist.barrier()
    ms = max_over_ranks(ms, dist)
    # The reference protocol redraws the multiplier while some right-hand side's residual
    # exceeds 1e-7 (genp.cpp:236-290); on this matrix the residuals straddle 1e-7, so a step
    # executes `attempts` full multiplier draws (G, A G, LU, solves, G Y).  The headline counts
    # the flops executed; value_per_solve counts one attempt's 1.4704e12.
    attempts = max(1, rep.attempts_drawn)
    cols = rl.last_column_reports(NRHS3)  # per right-hand side: the reference call's accepted draw
    value = world * attempts * FLOPS3 / (ms * 1e-3) / 1e12
    value_per_solve = world * FLOPS3 / (ms * 1e-3) / 1e12

    # backward error of the last solve, computed on the device (reported, not timed)
    res = (A @ X - B)
    bwd = float((res.norm(dim=0) / (A.norm() * X.norm(dim=0))).max())

    # dominant kernel: the A G DGEMM (2 n^3 flop per launch), timed alone on the same stream
    G = torch.empty(N3, N3, dtype=torch.float64, device=dev)
    AG = torch.empty_like(G)
    rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(SEED, 11 ^ 0x5000000000000000))
    for _ in range(2):
        rl.dev_gemm(A, G, AG)
    torch.cuda.synchronize()
    e0.record()
    reps = 5
    for _ in range(reps):
        rl.dev_gemm(A, G, AG)
    e1.record()
    torch.cuda.synchronize()
    gemm_ms = e0.elapsed_time(e1) / reps
    gemm_tf = 2 * N3 ** 3 / (gemm_ms * 1e-3) / 1e12
    # RNG stage alone (reported separately: not in the flop count)
    torch.cuda.synchronize()
    e0.record()
    rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(SEED, 11 ^ 0x5000000000000000))
    e1.record()
    torch.cuda.synchronize()
    rng_ms = e0.elapsed_time(e1)
    del G, AG

    # ---- e2e: public host-pointer call from pinned host memory ----
    L = rl.lib()
    L.rl_randomized_genp_ex.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                        C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p,
                                        C.c_void_p, C.c_uint32]
    L.rl_randomized_genp_ex.restype = C.c_int
    hA = A.cpu().pin_memory()
    hB = B.cpu().pin_memory()
    hX = torch.empty_like(hB).pin_memory()
    rl.lib().rl_set_stream(None)

    def step_e2e():
        st = L.rl_randomized_genp_ex(N3, NRHS3, hA.data_ptr(), hB.data_ptr(), 0, 0.0, 1.0, 1, 0, SEED, 11,
                                     hX.data_ptr(), None, 1)
        if st != 0:
            raise RuntimeError(rl.lib().rl_last_error().decode())

    step_e2e()
    if dist:
        dist.barrier()
    e2e_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_ms = max_over_ranks(e2e_ms, dist)
    e2e_value = world * attempts * FLOPS3 / (e2e_ms * 1e-3) / 1e12
    del hA, hB, hX

    # ---- config 2: batched n = 64 circulant +-1 (secondary line) ----
    # The 4096 systems are independent units: each rank solves its shard_range block (stream ids
    # stay the global system index + 7, so every system draws the same multiplier at any N).
    A2, b2, sids = make_config2_inputs(torch, dev, BATCH2)
    lo2, hi2 = shard_range(BATCH2, rank, world)
    A2, b2, sids = A2[lo2:hi2].contiguous(), b2[lo2:hi2].contiguous(), sids[lo2:hi2].contiguous()
    nsys2 = hi2 - lo2
    x2 = torch.empty_like(b2)
    ckind = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)

    def step2():
        rl.dev_randomized_genp_batched(A2, b2, x2, ckind, rl.MulSide.RIGHT, 0, SEED, sids)

    for _ in range(max(args.warmup, 3)):
        step2()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    k2 = max(args.steps, 10)
    e0.record()
    for _ in range(k2):
        step2()
    e1.record()
    torch.cuda.synchronize()
    ms2 = max_over_ranks(e0.elapsed_time(e1) / k2, dist)
    solves_s = BATCH2 / (ms2 * 1e-3)  # all ranks' systems over the max-over-ranks time
    res2 = torch.bmm(A2, x2.unsqueeze(2)).squeeze(2) - b2
    bwd2 = max_over_ranks(float((res2.norm(dim=1) / (A2.flatten(1).norm(dim=1) * x2.norm(dim=1))).max()), dist)
    fp64_frac2 = nsys2 * FLOPS2_PER_SYS / (ms2 * 1e-3) / 1e12 / fp64_peak  # per GPU
    hbm_frac2 = nsys2 * BYTES2_PER_SYS / (ms2 * 1e-3) / 1e9 / hbm_peak
    cpu2 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu2 = cpu_baseline_config2(A2[:256].cpu().numpy(), b2[:256].cpu().numpy())

    # ---- config 4: the randomized range finder (third line) ----
    rf = run_config4(torch, rl, dev, dist, rank, world, args, fp64_peak)
    # ---- configs 1 and 5 (latency-bound n = 256; n = 16384 with the new multipliers) ----
    c1 = run_config1(torch, rl, dev, dist, args, fp64_peak)
    c5 = None if args.skip_config5 else run_config5(torch, rl, dev, dist, args, fp64_peak, hbm_peak, rank, world)
    circ = run_circulant_fft(torch, rl, dev, dist, hbm_peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_config3(threads=1)

    prof = load_profile_traffic()
    traffic = prof.get("dgemm_dram_bytes_per_launch")
    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; reference RNG streams)",
        "config": config3(world),
        "run": {"attempts_per_step": attempts, "flop_per_step": attempts * FLOPS3,
                "value_per_solve_tflops": round(value_per_solve, 4),
                "backward_error_max": bwd, "residual": rep.residual,
                "attempt_worst_column": rep.attempt, "column_attempts": [c[0] for c in cols],
                "rng_ms_per_G": round(rng_ms, 3)},
        "roofline": {"bound": "tensor", "kernel": "k_dgemm_tm<128,64> (A G: TMA tensor copies + DMMA m8n8k4 f64)",
                     "achieved": round(gemm_tf, 3), "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
                     "frac": round(gemm_tf / fp64_peak, 4), "traffic": traffic,
                     "peak_source": "same-run FP64 DMMA probe (rl_probe_peaks; MEASURED_PEAKS.json has no fp64)",
                     "step_frac_of_fp64_peak": round(attempts * FLOPS3 / (ms * 1e-3) / 1e12 / fp64_peak, 4)},
        "e2e": {"value": round(e2e_value, 4), "unit": "TFLOP/s",
                "h2d_bytes_per_step": 8 * (N3 * N3 + N3 * NRHS3), "d2h_bytes_per_step": 8 * N3 * NRHS3,
                "ms_per_step": round(e2e_ms, 3), "call": "rl_randomized_genp_ex (host pointers, pinned)"},
        "gpu_launches": launches,
        "batched": {"workload": "config2: 4096 x n=64, circulant +-1, MulSide::Right, redraw protocol",
                    "scaling": "strong (4096 systems split by shard_range)", "systems_per_rank": nsys2,
                    "value": round(solves_s, 1), "unit": "solves/s", "ms_per_step": round(ms2, 4),
                    "backward_error_max": bwd2,
                    "roofline": {"bound": "fp64", "frac_fp64": round(fp64_frac2, 4),
                                 "frac_hbm": round(hbm_frac2, 4), "peak_fp64": round(fp64_peak, 3),
                                 "peak_hbm_gbs": round(hbm_peak, 1)},
                    "cpu_baseline": cpu2},
        "range_finder": rf,
        "config1": c1,
        "config5": c5,
        "circulant_fft": circ,
        "clocks": clocks.summary(),
        "peaks_same_run": {"fp64_dmma_tflops": round(fp64_peak, 3), "hbm_copy_gbs": round(hbm_peak, 1)},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    return line


# ------------------------------------------------------- CPU baseline legs ----
def cpu_baseline_config3(threads: int = 1):
    """The reference's own CPU code (oracle/_ref, compiled from /root/reference) on a bounded
    sample of the config-3 work: Matrix::multiply of a row slab of A (rows split over
    `threads` threads, each a reference call) against the full 8192^2 G, plus one genp_factor
    (the reference's LU is single-threaded) at n = 1024.  value = sample flop / sample time."""
    from oracle.pyoracle import Reference, Restated
    kind = "reference" if Reference.available() else "port"
    lib = Reference() if kind == "reference" else Restated()
    rng = np.random.default_rng(0)
    G = rng.standard_normal((N3, N3))
    rows_per = 8
    slabs = [rng.standard_normal((rows_per, N3)) for _ in range(threads)]
    t0 = time.perf_counter()
    ts = [threading.Thread(target=lib.matmul, args=(s, G)) for s in slabs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    t_mm = time.perf_counter() - t0
    f_mm = 2.0 * rows_per * threads * N3 * N3
    nl = 1024
    M = rng.standard_normal((nl, nl)) + nl * np.eye(nl)
    t0 = time.perf_counter()
    lib.genp_factor(M, 0.0)
    t_lu = time.perf_counter() - t0
    f_lu = 2.0 * nl ** 3 / 3
    value = (f_mm + f_lu) / (t_mm + t_lu) / 1e12
    return {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": kind,
            "sample": f"Matrix::multiply {rows_per * threads}x{N3} slab x {N3}^2 G ({threads} thread(s)) "
                      f"+ genp_factor n={nl} (1 thread); {t_mm + t_lu:.2f} s",
            "host": _host_cpu()}


def _ref_lib():
    from oracle.pyoracle import Reference, Restated
    kind = "reference" if Reference.available() else "port"
    return kind, (Reference() if kind == "reference" else Restated())


def cpu_baseline_config1(A, b):
    """The reference's randomized_genp (Gaussian, Right, refine 0; its contrast arm included,
    as the reference always runs it) on the config-1 system, 1 thread: us per solve."""
    kind, lib = _ref_lib()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        lib.randomized_genp(A, b, "gaussian", "right", 0, seed=SEED, sid=15)
    us = (time.perf_counter() - t0) * 1e6 / reps
    return {"value": round(us, 1), "unit": "us/solve", "cores": 1, "kind": kind,
            "sample": f"randomized_genp n=256 x {reps} (contrast arm included)"}


def cpu_baseline_config2(A, b, nsys: int = 256):
    """The reference's randomized_genp (CirculantSign, Right) per system, as table1_genp loops it,
    on the first `nsys` config-2 systems: 1 thread and all host threads (solves/s)."""
    kind, lib = _ref_lib()

    def run(lo, hi):
        for t in range(lo, hi):
            lib.randomized_genp(A[t], b[t], "circulant_sign", "right", 0, seed=SEED, sid=7 + t)
    t0 = time.perf_counter()
    run(0, nsys)
    one = nsys / (time.perf_counter() - t0)
    th = os.cpu_count() or 1
    chunks = [(i * nsys // th, (i + 1) * nsys // th) for i in range(th)]
    t0 = time.perf_counter()
    ts = [threading.Thread(target=run, args=c) for c in chunks]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    allc = nsys / (time.perf_counter() - t0)
    return {"value": round(allc, 1), "unit": "solves/s", "cores": th, "kind": kind,
            "value_1_thread": round(one, 1),
            "sample": f"{nsys} systems, randomized_genp per system (contrast arm included)"}


def cpu_baseline_config4(A_slab, H):
    """The reference's Matrix::multiply for Y = A H on a row slab of the config-4 A (the
    dominant CPU cost; the QR and SVD are Eigen in the reference and not compiled here):
    TFLOP/s, 1 thread."""
    kind, lib = _ref_lib()
    t0 = time.perf_counter()
    lib.matmul(A_slab, H)
    dt = time.perf_counter() - t0
    fl = 2.0 * A_slab.shape[0] * A_slab.shape[1] * H.shape[1]
    return {"value": round(fl / dt / 1e12, 6), "unit": "TFLOP/s", "cores": 1, "kind": kind,
            "sample": f"Matrix::multiply {A_slab.shape[0]}x{A_slab.shape[1]} slab x H {H.shape[0]}x{H.shape[1]}; "
                      f"{dt:.2f} s"}


def cpu_baseline_config5(A_host, threads: int):
    """Config 5's CPU arms on bounded samples: the reference's Gaussian
    arm = Matrix::multiply of a row slab of A against the 16384^2 G (all host threads, one
    reference call per thread) + genp_factor at n = 1024 (single-threaded in the reference);
    the Householder-pair and sparse +-1 applies through the C restatement (oracle/rl_oracle.c,
    the reference has no such multipliers) on the full 16384^2 A, 1 thread (GB/s over the same
    algorithmic bytes as the GPU kernels: 2 n^2 8)."""
    from oracle.pyoracle import Restated
    kind, lib = _ref_lib()
    n = A_host.shape[0]
    rng = np.random.default_rng(5)
    G = rng.standard_normal((n, n))
    rows_per = 4
    slabs = [np.ascontiguousarray(A_host[i * rows_per:(i + 1) * rows_per]) for i in range(threads)]
    t0 = time.perf_counter()
    ts = [threading.Thread(target=lib.matmul, args=(sl, G)) for sl in slabs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    t_mm = time.perf_counter() - t0
    del G
    nl = 1024
    M = rng.standard_normal((nl, nl)) + nl * np.eye(nl)
    t0 = time.perf_counter()
    lib.genp_factor(M, 0.0)
    t_lu = time.perf_counter() - t0
    f = 2.0 * rows_per * threads * n * n + 2.0 * nl ** 3 / 3
    gauss = {"value": round(f / (t_mm + t_lu) / 1e12, 6), "unit": "TFLOP/s", "cores": threads, "kind": kind,
             "sample": f"Matrix::multiply {rows_per * threads}x{n} slab x {n}^2 G ({threads} threads) + "
                       f"genp_factor n={nl} (1 thread); {t_mm + t_lu:.2f} s"}
    O = Restated()
    u1, u2 = O.householder_pair_signs(n, SEED, 55)
    rows, signs = O.sparse_pm1(n, SEED, 56)
    bytes_ = 2.0 * n * n * 8
    t0 = time.perf_counter()
    O.hh2_apply_right(u1, u2, A_host)
    t_hh = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.sparse_apply_right(rows, signs, A_host)
    t_sp = time.perf_counter() - t0
    return {"gaussian": gauss,
            "householder_pair": {"value": round(bytes_ / t_hh / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
                                 "sample": f"A H1 H2 on the full {n}^2 A (rlo_hh2_apply_right); {t_hh:.2f} s"},
            "sparse_sign": {"value": round(bytes_ / t_sp / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
                            "sample": f"A S on the full {n}^2 A (rlo_sparse_apply_right); {t_sp:.2f} s"}}


def _host_cpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), "?")
    except OSError:
        model = "?"
    return {"nproc": os.cpu_count(), "model": model}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation of the path on the host cores."""
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_baseline_config3(threads)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline_config3(threads))
    wall = time.perf_counter() - t0
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config3(world),
            "sample_note": "each step is a bounded sample of the config-3 work on the host cores (cpu_baseline.sample)",
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-config5", action="store_true", help="skip the n = 16384 config-5 arms (~10 s)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, dist, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
