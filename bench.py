#!/usr/bin/env python
"""bench.py -- hybrid LDU factor + Schur (Alg. 1 of arXiv 2208.01907) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl hf|reference]

One STEP = one pass of the whole hot path over one
synthetic matrix already resident in HBM:
    restore Kbar (D2D copy, the scaling is in place) -> hf_scale ->
    hf_factor_lowprec -> hf_schur_gcr -> hf_factor_hard
Inputs are larger than L2 (K is 2.1 GB at C2), so no L2 flush is needed.
The metric is BASELINE.json's "hybrid LDU factor+Schur time (s), TFLOP/s":
value = algorithmic TFLOP/s of the whole job (DESIGN.md section 7 gives the
flop model), with seconds per factorization alongside.

N > 1 (torchrun): replicas -- every rank factorises its own seeded matrix, no
data-path collective; weak scaling, max-over-ranks time.

--impl reference: the CPU oracle (oracle/, plain C + numpy) timed on the
host cores on a bounded sample of the same workload (rank 0 only).
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

FFMA_PEAK_DERIVED = 148 * 128 * 2 * 1.965e9 / 1e12     # TFLOP/s, B200 FP32 non-tensor
DMMA_PEAK_MEASURED = 37.15                              # tools/peaks.py, profiles/peaks_r01.json
KCLASSES = ("scale", "chain", "trailing", "dgemm", "trsm", "trsm_setup", "gram", "hard", "other",
            "ozaki_split", "ozaki_imma", "ozaki_combine")
OZAKI_SLICES = 8                                        # ozaki.cu default (hf_gcr_opts.slices = 0)
OZAKI_MODULI = 16                                       # ozaki2.cu (the residue form)


def int8_peak():
    """Dense int8 tensor peak: the driver-measured bf16 dense peak (MEASURED_PEAKS.json,
    burst) x the nominal int8 / bf16 ratio (4.5 / 2.25 POPS, B200_PROFILING.md)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        return 2.0 * bf16, "MEASURED_PEAKS.json bf16_tflops (burst) x 2 (nominal int8 / bf16 ratio)"
    except Exception:
        return 4500.0, "nominal B200 dense int8 (no MEASURED_PEAKS.json)"


def flop_model(L, N, Ntau, n2, iters, ozaki=False):
    """Algorithmic flops of one hybrid factorization, counted
    as block_gcr (gcr.cu) runs Alg. 5: K11-products for r_0, q_0, each z_{n+1} of a
    non-final iteration and the reported true residual (iters + 2); preconditioner
    applications for x_0, w_0 and each w_{n+1} of a non-final iteration (iters + 1);
    per iteration M_n, A_n, the X and R updates (4 N x n2 x n2 products) and, on a
    non-final iteration n, Q_m^T z and the P, Q updates over the n + 1 blocks
    (3 (n + 1) products) plus the n2 x n2 products C = M^-1 A and G_m."""
    m = np.arange(L, L - Ntau, -1, dtype=np.float64)          # active size before each pivot
    f1 = float(np.sum((m - 1.0) * m))                          # rank-1 updates of the lower triangle
    mv = 2.0 * N * N * n2                                      # K11 W
    pc = 2.0 * N * N * n2                                      # FP32 fwd + bwd triangular solves
    nn = 2.0 * N * n2 * n2
    gram = sum(nn * 4 for n in range(iters)) + sum(nn * 3 * (n + 1) for n in range(iters - 1))
    small = 2.0 * n2 ** 3 * (iters + sum(n + 1 for n in range(iters - 1)))
    f2 = (iters + 2) * mv + (iters + 1) * pc + gram + small
    f3 = 2.0 * N * n2 * n2
    f4 = n2 ** 3 / 3.0
    matvec = (iters + 2) * mv
    dmma = (0.0 if ozaki else matvec) + gram + small + f3      # the FP64 DMMA GEMM class
    return {"stage1": f1, "gcr": f2, "schur": f3, "hard": f4, "total": f1 + f2 + f3 + f4,
            "dmma": dmma, "matvec": matvec, "trsm": (iters + 1) * pc}


def trsm_roofline(N, n2, iters, flops, ms, setup_ms, ach, nbytes):
    """The FP32 preconditioner's roofline.  Default form (k_trsm_blk.cu): blocked solves whose
    products run on the bf16 tensor cores as six exact-part products each (FP32 precision);
    its executed bf16 work per application is 6 x (the diagonal-block inverse products + the
    off-diagonal updates) x 2 directions on the padded size Nb = nb BS, BS = 2048 (the
    k_trsm_blk.cu rule), against the measured bf16 peak; the FP32-equivalent rate is
    reported against the FFMA peak.  HF_PRECOND=dataflow: the FFMA2 dataflow kernels."""
    if os.environ.get("HF_PRECOND") == "dataflow":
        return {"kernel": "k_trsm<fwd/bwd> (FP32 FFMA2 dataflow triangular solves, n2 right-hand sides)",
                "bound": "alu", "achieved": ach, "peak": FFMA_PEAK_DERIVED, "unit": "TFLOP/s",
                "frac": ach / FFMA_PEAK_DERIVED if ach else None, "flops_per_step": flops, "ms_per_step": ms,
                "hbm_gbs": nbytes / (ms * 1e-3) / 1e9 if ms > 0 else None, "setup_ms_per_step": setup_ms}
    BS = 64
    while BS < 2048 and BS < N:
        BS *= 2
    nb = -(-N // BS)
    Nb = nb * BS
    ncp = -(-n2 // 8) * 8
    per_dir = nb * 2.0 * BS * BS * ncp + sum(2.0 * (Nb - (j + 1) * BS) * BS * ncp for j in range(nb - 1))
    bf16_fl = 6 * 2 * per_dir * (iters + 1)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bpk, src = float(json.load(f)["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (burst)"
    except Exception:
        bpk, src = 2250.0, "nominal B200 dense bf16"
    b_ach = bf16_fl / (ms * 1e-3) / 1e12 if ms > 0 else None
    return {"kernel": "blocked FP32 preconditioner (k_trsm_blk.cu: %d-row diagonal-block inverses + "
                      "off-diagonal updates, each product as 6 exact bf16-part GEMMs on cuBLASLt, FP32 "
                      "accumulation; k_blk_split_rows / gather / dscale / scatter)" % BS,
            "bound": "bf16_tensor", "achieved": b_ach, "peak": bpk, "unit": "TFLOP/s",
            "frac": b_ach / bpk if b_ach else None, "peak_source": src, "bf16_flops_per_step": bf16_fl,
            "fp32_equivalent_tflops": ach, "fp32_equivalent_vs_ffma_peak": ach / FFMA_PEAK_DERIVED if ach else None,
            "flops_per_step": flops, "ms_per_step": ms, "block_rows": BS, "blocks": nb,
            # per application and direction: nb inverse products, nb - 1 couplings (one GEMM each
            # over K' = 6 BS) and three bulk GEMMs for each of nb - 2 blocks; the setup's doubling
            # levels (2 each) and the 12 batched coupling part products
            "library_launches_per_step": (iters + 1) * 2 * (nb + (nb - 1) + 3 * max(nb - 2, 0))
                                         + 2 * max(0, int(np.log2(BS // 64))) + (12 if nb > 1 else 0),
            "hbm_gbs": nbytes / (ms * 1e-3) / 1e9 if ms > 0 else None, "setup_ms_per_step": setup_ms}


class Clocks:
    """Clock / throttle-reason sampler for the timed region.  NVML in-process
    (the same counters nvidia-smi's clocks line reads: clocks.sm, clocks.max.sm,
    power.draw, clocks_event_reasons.*), every 200 ms; a subprocess per sample
    would perturb the host-driven parts of the step it is measuring.  Falls
    back to nvidia-smi if NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0, enabled=True):
        self.index, self.samples, self.stop, self.enabled = index, [], threading.Event(), enabled
        self.th = threading.Thread(target=self._run, daemon=True)
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nv = None
        try:                     # the first queries are slow (NVML warm-up): keep them out of the timed region
            for _ in range(3):
                self._sample()
        except Exception:
            pass

    def _sample(self):
        if self.nv is not None:
            nv, h = self.nv, self.h
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            return [nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                    nv.nvmlDeviceGetPowerUsage(h) / 1e3] + [bool(r & b_) for b_ in bits]
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        r = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", str(self.index)],
                           capture_output=True, text=True, timeout=5)
        v = [x.strip() for x in r.stdout.strip().split(",")]
        return [float(v[0]), float(v[1]), float(v[2])] + [x.lower() == "active" for x in v[3:7]]

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        if self.enabled:
            self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.enabled:
            self.th.join(timeout=10)

    def summary(self):
        mhz = [s[0] for s in self.samples]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(self.NAMES, s[3:7]):
                if v:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(mhz)) if mhz else None,
                "sm_max_mhz": float(self.samples[-1][1]) if self.samples else None,
                "power_w_max": float(max(s[2] for s in self.samples)) if self.samples else None,
                "reasons": sorted(reasons), "samples": len(mhz),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def load_traffic():
    """Per-launch DRAM bytes of the roofline kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU oracle sample
def oracle_sample(Kb_np, spec, pivots=1024):
    """The oracle as it stands on a bounded sample of the same workload:
    its stage 1 for the first `pivots` pivots of the config's matrix, plus one
    block-GCR iteration's FP64 mat-vec and FP32 preconditioner solves at the
    config's sizes.  Returns (flops, seconds, description)."""
    import oracle
    L = Kb_np.shape[0]
    t0 = time.perf_counter()
    K, q = oracle.scale(Kb_np)
    t1 = time.perf_counter()
    F = oracle.factor_lowprec(K, spec.tau, n_min=spec.n_min, max_steps=pivots)
    t2 = time.perf_counter()
    done = F.Ntau
    m = np.arange(L, L - done, -1, dtype=np.float64)
    f_st1 = float(np.sum((m - 1.0) * m))
    # one GCR iteration worth of oracle kernels on operands of the config's sizes
    n2 = max(spec.n_min, 4)
    N = L - n2
    rng = np.random.default_rng(0)
    W = rng.standard_normal((N, n2))
    Lf = np.tril(rng.standard_normal((N, N)).astype(np.float32) * (1.0 / N), -1) + np.eye(N, dtype=np.float32)
    Fs = oracle.LowFactor(L=N, N=N, Ntau=N, perm=np.arange(N), D=np.ones(N, np.float32),
                          Lfac=np.asfortranarray(Lf), dtype=np.float32)
    K11 = K[:N, :N]
    t3 = time.perf_counter()
    Z = K11 @ W
    E = oracle.precond_apply(Fs, Z)
    t4 = time.perf_counter()
    del E
    f_it = 2.0 * N * N * n2 * 2
    secs = (t1 - t0) + (t2 - t1) + (t4 - t3)
    desc = (f"oracle scale + stage 1 (first {done} pivots of {spec.name}, L={L}) + one block-GCR "
            f"iteration's K11 W and FP32 preconditioner at N={N}, n2={n2}")
    return f_st1 + f_it, secs, desc


def oracle_full(Kb_np, spec):
    """The WHOLE oracle (Alg. 1 steps 1-5: scale, stage 1, block GCR, Schur, hard
    factorization) on the config's matrix, as it stands.  Returns (flops, seconds,
    description) with the same flop model as the GPU line."""
    import oracle
    L = Kb_np.shape[0]
    t0 = time.perf_counter()
    K, _ = oracle.scale(Kb_np)
    HF = oracle.hybrid_factor(K, tau=spec.tau, n_min=spec.n_min)
    secs = time.perf_counter() - t0
    fm = flop_model(L, HF.F.N, HF.F.Ntau, HF.F.n2, HF.gcr.iters)
    desc = (f"the whole oracle on {spec.name} (L={L}): scale + FP32 stage 1 + block GCR "
            f"({HF.gcr.iters} iterations, n2={HF.F.n2}) + Schur + hard factorization")
    return fm["total"], secs, desc


def max_over_ranks(x: float) -> float:
    """Max of a per-rank scalar over the default process group (NCCL: device
    tensor, gloo: host tensor); identity without a group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    """Sum of a per-rank scalar over the default process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def spawn_ranks(n: int) -> None:
    """bench.py --gpus N without WORLD_SIZE: run N ranks under torch.distributed.run
    on 127.0.0.1 (the contract's launch) and pass their output through."""
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    if r.returncode != 0:
        raise SystemExit(r.returncode)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="hf", choices=["hf", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pivots-sample", type=int, default=1024)
    ap.add_argument("--cpu-baseline", default="auto", choices=["auto", "full", "sample", "none"],
                    help="auto: the whole oracle when L <= 16384 (C2: ~2 min on 16 host cores), else the "
                         "bounded sample")
    ap.add_argument("--mode", default=None, choices=["replicas", "shard"],
                    help="N>1 (default shard): shard = ONE matrix factored by all ranks -- stage 1 "
                         "distributed (lower-triangle 1D block-cyclic, per-pivot key exchange over NVLink), "
                         "block-GCR right-hand sides split over the ranks with the S22 / X12 slices broadcast "
                         "(strong scaling); replicas = one matrix per rank, no data-path collective (weak)")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None and args.impl == "hf":
        # launch our own ranks (one process per GPU) and relay rank 0's line
        return spawn_ranks(args.gpus)
    if world_env is not None and args.impl == "hf" and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.mode is None:
        args.mode = "shard" if args.gpus > 1 else "replicas"
    if args.config is None:
        # N = 1: the configuration the single-GPU targets are quoted on (C2); N > 1: the
        # scale-out configuration (C4, L = 65536) factored across the ranks
        args.config = "C4" if (args.gpus > 1 and args.mode == "shard") else "C2"

    import torch
    import torch.distributed as dist

    import hf_inputs as hi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec = hi.CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        Kb = hi.make_kbar(spec, args.seed, device="cuda" if (torch.cuda.is_available() and spec.L > 4096) else "cpu")
        if spec.L > 16384:
            # a bounded sample of the scale-out workload: its leading 16384 x 16384 principal
            # block (the same planted construction), so every step stays within seconds
            Kb = Kb[:16384, :16384].contiguous()
        Kb = Kb.cpu().numpy()
        for _ in range(args.warmup):
            oracle_sample(Kb, spec, pivots=max(16, args.pivots_sample // 16))
        fl, sec = 0.0, 0.0
        desc = ""
        for _ in range(args.steps):
            f, s_, desc = oracle_sample(Kb, spec, pivots=args.pivots_sample // 4)
            fl += f
            sec += s_
        v = fl / sec / 1e12
        line = {"metric": "hybrid_factor_schur_tflops", "value": v, "unit": "TFLOP/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": sec / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "fp32+fp64", "data": "synthetic",
                "config": {"workload": spec.name, "L": spec.L, "tau": spec.tau, "n_min": spec.n_min,
                           "seed": args.seed, "parallelism": "none (host cores)"},
                "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": host_cores(), "kind": "oracle",
                                 "sample": desc},
                "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    from paper_2208_01907_b200 import hf

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    if args.mode == "shard" and world > 1:
        idb = [hf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idb, src=0)
        ctx = hf.Context(local, stream, nccl_id=idb[0], rank=rank, nranks=world)
    else:
        ctx = hf.Context(local, stream)

    # ---- the workload (seeded, synthetic; each rank its own seed in replica mode)
    gen_dev = "cuda" if spec.L > 4096 else "cpu"
    seed = args.seed + (rank if args.mode == "replicas" else 0)
    Kb = hi.make_kbar(spec, seed, device=gen_dev).to(dev).contiguous()
    if dev.type == "cuda":
        # the generator's temporaries stay in torch's cache (C4: 39 GB beside the 34 GB input),
        # which the library's device memory (the int8 residues of K) then cannot use
        torch.cuda.empty_cache()
    # L > 32768 (C4, 34 GB in FP64): no pristine device copy -- every step scales K in
    # place; after the first, hf_scale sees an already-scaled matrix (Q = I, the same
    # bits) and does the same reads, multiplications and writes
    restore = spec.L <= 32768
    K = torch.empty_like(Kb) if restore else Kb
    torch.cuda.synchronize()

    def step(profile=False):
        if restore:
            K.copy_(Kb)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        hf.hf_scale(ctx, K)
        ev[1].record(stream)
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
        ev[2].record(stream)
        hy, info, _ = hf.hf_schur_gcr(ctx, K, lf)
        ev[3].record(stream)
        kd = hf.hf_factor_hard(ctx, hy)
        ev[4].record(stream)
        res = (lf.N, lf.L - lf.n2_tau_only, lf.n2, info.iters, kd, info.max_rel_res_true, info.matvec)
        hy.close()               # one factorization's buffers live at a time: the library's
        lf.close()               # memory cache then serves every step from the same blocks
        return res, ev

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if os.environ.get("HF_ALLOC_DEBUG"):
        print("[bench] warm-up done", file=sys.stderr, flush=True)

    ctx.set_profiling(True)
    for c in KCLASSES:
        ctx.kernel_stats(c)            # drain the warm-up records
    base = {c: ctx.kernel_stats(c) for c in KCLASSES}
    wbase = {c: ctx.kernel_work(c) for c in KCLASSES}
    launches0 = ctx.launch_count()
    stage_ms = np.zeros(4)
    step_ms = []
    results = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.disable()              # no collector pauses inside the timed region
    with Clocks(local, enabled=not os.environ.get("HF_BENCH_NO_CLOCKS")) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            res, ev = step()
            results.append(res)
            for q in range(4):
                stage_ms[q] += ev[q].elapsed_time(ev[q + 1]) if ev[q + 1].query() else 0.0
            step_ms.append([round(ev[q].elapsed_time(ev[q + 1]), 2) for q in range(4)])
        t_end.record(stream)
        torch.cuda.synchronize()
    gc.enable()
    if world > 1:
        dist.barrier()
    elapsed = t_start.elapsed_time(t_end)             # ms, this rank
    launches = ctx.launch_count() - launches0
    ctx.set_profiling(False)
    kstats = {c: ctx.kernel_stats(c) for c in base}
    kms = {c: (kstats[c][0] - base[c][0]) / args.steps for c in base}
    klaunch = {c: (kstats[c][1] - base[c][1]) / args.steps for c in base}
    kwork = {c: tuple((a - b) / args.steps for a, b in zip(ctx.kernel_work(c), wbase[c])) for c in base}

    N, Ntau, n2, iters, kd, tres, mv_form = results[-1]
    L = spec.L
    ozaki = kms.get("ozaki_imma", 0.0) > 0.0
    fm = flop_model(L, N, Ntau, n2, iters, ozaki=ozaki)
    elapsed = max_over_ranks(elapsed)
    ms_step = elapsed / args.steps
    # replicas: every rank factorises its own matrix (weak scaling); shard: one
    # factorization per step with stage 2 split over the ranks (strong scaling)
    # (replicas: each rank's own matrix and iteration count, summed over the ranks)
    total_flops = sum_over_ranks(fm["total"]) if args.mode == "replicas" else fm["total"]
    value = total_flops / (ms_step * 1e-3) / 1e12

    # ---- roofline of the dominant compute kernel (the FP32 trailing update): its OWN
    # algorithmic flops (one FMA per lower-triangle entry per pivot of each launch, as
    # libhf reports them per launch; the in-panel part of F1 is the chain's)
    tr_ms = kms["trailing"]
    tr_fl = kwork["trailing"][0]
    achieved = tr_fl / (tr_ms * 1e-3) / 1e12 if tr_ms > 0 else None
    traffic = load_traffic()
    roof = {"kernel": "k_trailing_c (FP32 FFMA2 symmetric rank-nb update, bitwise canonical order)",
            "bound": "alu", "achieved": achieved, "peak": FFMA_PEAK_DERIVED, "unit": "TFLOP/s",
            "frac": (achieved / FFMA_PEAK_DERIVED) if achieved else None,
            "peak_source": "derived 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md sec. 7); "
                           "microbenchmark 72.6 FFMA / 74.3 FFMA2 TF/s (profiles/peaks_r01.json)",
            "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "traffic_note": traffic.get("note") if traffic else "no ncu capture committed yet",
            "flops_per_step": tr_fl, "ms_per_step": tr_ms, "launches_per_step": klaunch["trailing"]}
    # ---- the chain's floor: its grid-wide exchange alone, in the geometry libhf picks
    # (k_lowprec.cu: max(64, L / rows-that-fit) CTAs, at most one per SM; one thread per row)
    xfloor = None
    if world == 1 or args.mode == "replicas":
        try:
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            g_ct = min(nsm, max(64, -(-L // 358)), max(1, -(-L // 32)))
            xfloor = ctx.chain_exchange_floor(g_ct, -(-(-(-L // g_ct)) // 32) * 32, 8192)
        except Exception:
            xfloor = None
    # ---- the other kernels' own rooflines
    dg_ms, ts_ms, ch_ms = kms["dgemm"], kms["trsm"], kms["chain"]
    dmma_ach = fm["dmma"] / (dg_ms * 1e-3) / 1e12 if dg_ms > 0 else None
    trsm_ach = kwork["trsm"][0] / (ts_ms * 1e-3) / 1e12 if ts_ms > 0 else None
    rooflines = {
        "dgemm": {"kernel": ("k_dgemm (FP64 DMMA mma.sync m8n8k4: Gram / update products, Schur; the K11 W "
                             "mat-vecs run on the int8 tensor cores, rooflines.matvec)") if ozaki else
                            "k_dgemm (FP64 DMMA mma.sync m8n8k4: K11 W mat-vecs, Gram / update products, Schur)",
                  "bound": "fp64_tensor", "achieved": dmma_ach, "peak": DMMA_PEAK_MEASURED, "unit": "TFLOP/s",
                  "frac": dmma_ach / DMMA_PEAK_MEASURED if dmma_ach else None,
                  "flops_per_step": fm["dmma"], "flops_note": "algorithmic DMMA work only (%sGram / update / "
                  "n2 x n2 products, S22); the FP32 preconditioner is not in it" %
                  ("" if ozaki else "mat-vecs on N = |Lambda_1| rows, "),
                  "executed_flops_per_step": kwork["dgemm"][0], "ms_per_step": dg_ms,
                  "peak_source": "measured DMMA microbenchmark (tools/peaks.py, profiles/peaks_r01.json)"},
        "trsm": trsm_roofline(N, n2, iters, kwork["trsm"][0], ts_ms, kms["trsm_setup"], trsm_ach,
                              kwork["trsm"][1]),
        "chain": {"kernel": "k_chain (cooperative persistent pivot chain, one launch per panel)",
                  "bound": "latency", "us_per_pivot": ch_ms * 1e3 / max(Ntau, 1), "ms_per_step": ch_ms,
                  "exchange_floor_us": xfloor, "frac_of_floor": (xfloor / (ch_ms * 1e3 / max(Ntau, 1)))
                  if (xfloor and ch_ms > 0) else None,
                  "floor_note": "the chain's grid-wide exchange alone (hf_chain_exchange_floor: block key "
                                "reduction + tagged slot store + poll of every slot, same CTA geometry, no column "
                                "fetch, no arithmetic), measured live after the timed region",
                  "hbm_gbs": kwork["chain"][1] / (ch_ms * 1e-3) / 1e9 if ch_ms > 0 else None,
                  "bytes_per_step": kwork["chain"][1]},
    }
    if ozaki:
        # the FP64 mat-vec emulated on the int8 tensor cores (ozaki.cu): s(s+1)/2 exact slice
        # products per mat-vec, each 2 N^2 n2 int8 ops of algorithmic work; the int8 GEMMs are
        # cuBLASLt's (a plain library GEMM), the splitting and the combination libhf's
        mv_ms = kms["ozaki_split"] + kms["ozaki_imma"] + kms["ozaki_combine"]
        crt = mv_form == 3
        nprod = OZAKI_MODULI if crt else OZAKI_SLICES * (OZAKI_SLICES + 1) // 2
        i8_ops = nprod * fm["matvec"]
        i8_peak, i8_src = int8_peak()
        i8_ach = i8_ops / (kms["ozaki_imma"] * 1e-3) / 1e12
        rooflines["matvec"] = {
            "kernel": ("K11 W as FP64 emulated on the int8 tensor cores, residue (CRT) form: 53-bit integer "
                       "scalings, %d moduli <= 256 (k_oz2_residues, %d exact int8 GEMMs per mat-vec on cuBLASLt "
                       "IMMA as one strided batch, k_oz2_combine: Garner mixed radix + FP64 Horner)" % (OZAKI_MODULI, OZAKI_MODULI)) if crt
                      else ("K11 W as FP64 emulated on the int8 tensor cores (Ozaki scheme, %d slices: k_oz_split, "
                            "%d int8 GEMMs per mat-vec on cuBLASLt IMMA, k_oz_combine<%d>)" %
                            (OZAKI_SLICES, OZAKI_SLICES, OZAKI_SLICES)),
            "bound": "int8_tensor", "achieved": i8_ach, "peak": i8_peak, "unit": "TOP/s", "frac": i8_ach / i8_peak,
            "peak_source": i8_src, "int8_ops_per_step": i8_ops, "products_per_matvec": nprod,
            "fp64_equivalent_tflops": fm["matvec"] / (mv_ms * 1e-3) / 1e12,
            "fp64_equivalent_vs_dmma_peak": fm["matvec"] / (mv_ms * 1e-3) / 1e12 / DMMA_PEAK_MEASURED,
            "ms_per_step": mv_ms, "imma_ms_per_step": kms["ozaki_imma"], "split_ms_per_step": kms["ozaki_split"],
            "combine_ms_per_step": kms["ozaki_combine"],
            "library_launches_per_step": (iters + 2) * (1 if crt else OZAKI_SLICES)}
    shares = {c: round(kms[c] / ms_step, 4) for c in kms}

    line = {"metric": "hybrid_factor_schur_tflops", "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if args.mode == "replicas" else "strong", "vs_baseline": None,
            "dtype": "fp32+fp64+i8" if ozaki else "fp32+fp64", "data": "synthetic",
            "matvec_form": {1: "fp64 DMMA", 2: "int8 slices (Ozaki)", 3: "int8 residues (CRT)"}.get(mv_form),
            "config": {"workload": spec.name, "L": L, "N": N, "n2": n2, "n2_tau_only": L - Ntau,
                       "tau": spec.tau, "n_min": spec.n_min, "seed": args.seed, "gcr_iters": iters,
                       "kernel_dim": kd, "gcr_true_rel_res": tres,
                       "parallelism": ("single" if world == 1 else
                                       ("replicas" if args.mode == "replicas" else
                                        f"stage1-dist{world} (lower-triangle 1D block-cyclic) + stage2-rhs-shard{world}")),
                       "l2": "inputs larger than L2 (K fp64 %.2f GB); %s" %
                             (8 * L * L / 1e9, "restore copy of Kbar inside each step" if restore else
                              "K scaled in place every step (idempotent after the first)")},
            "seconds_per_factorization": ms_step / 1e3,
            "stage_ms": {"scale": stage_ms[0] / args.steps, "lowprec": stage_ms[1] / args.steps,
                         "schur_gcr": stage_ms[2] / args.steps, "hard": stage_ms[3] / args.steps},
            "flops_per_step": fm, "per_step_stage_ms": step_ms,
            "kernel_ms_per_step": kms, "kernel_share": shares,
            "chain_us_per_pivot": kms["chain"] * 1e3 / max(Ntau, 1),
            "dgemm_tflops": dmma_ach,
            "roofline": roof, "rooflines": rooflines, "gpu_launches": int(launches), "clocks": clk.summary()}

    # ---- end to end through the public API with host buffers
    if not args.no_e2e:
        ser_ms = None
        try:
            Kh = (Kb if restore else hi.make_kbar(spec, seed, device=gen_dev)).cpu().pin_memory()
            e2e_steps = max(1, args.steps) if restore else 1   # C4: 34 GB per rank crosses the host link once
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            # double-buffered input: step s+1's matrix crosses the host link (its lower
            # triangle, the only part the scaling reads; the device mirrors it) on the
            # library's upload stream while step s factors
            Kd = [K] + ([torch.empty_like(K)] if e2e_steps > 1 else [])
            d2h = 0
            h2d = hf.hf_upload_lower(ctx, Kh, Kd[0])
            for s_ in range(e2e_steps):
                Ks = Kd[s_ % len(Kd)]
                hf.hf_scale(ctx, Ks)   # ordered after this step's upload; the stream is idle after it
                if s_ + 1 < e2e_steps:
                    hf.hf_upload_lower(ctx, Kh, Kd[(s_ + 1) % len(Kd)])
                K_ = Ks
                lf = hf.hf_factor_lowprec(ctx, K_, tau=spec.tau, n_min=spec.n_min)
                hy, info, S22 = hf.hf_schur_gcr(ctx, K_, lf, want_S22_host=True)
                kd = hf.hf_factor_hard(ctx, hy)
                perm, D, _ = lf.export(with_L=False)
                d2h = S22.nbytes if S22 is not None else 0
                d2h += perm.nbytes + D.nbytes + 8
                hy.close()
                lf.close()
            t1.record(stream)
            torch.cuda.synchronize()
            e_ms = t0.elapsed_time(t1) / e2e_steps
            # the same steps with the copy NOT overlapped (hf_scale_host: copy, then scale, then
            # the factorization), reported beside the pipelined figure
            ser_steps = min(3, e2e_steps) if restore else 0
            if ser_steps:
                t2 = torch.cuda.Event(enable_timing=True)
                t3 = torch.cuda.Event(enable_timing=True)
                t2.record(stream)
                for _ in range(ser_steps):
                    hf.hf_scale_host(ctx, Kh, K)
                    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
                    hy, info, S22 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True)
                    hf.hf_factor_hard(ctx, hy)
                    lf.export(with_L=False)
                    hy.close()
                    lf.close()
                t3.record(stream)
                torch.cuda.synchronize()
                ser_ms = t2.elapsed_time(t3) / ser_steps
            e2e_err = None
        except Exception as e:   # a failed end-to-end leg must not lose the device-timed line
            e_ms, e2e_err = -1.0, repr(e)[:300]
        e_ms = max_over_ranks(e_ms)   # every rank takes part, failed or not
        ser_ms = max_over_ranks(ser_ms if ser_ms else -1.0)
        if e2e_err is None and e_ms > 0:
            line["e2e"] = {"value": total_flops / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                           "ms_per_step": e_ms,
                           "unpipelined_ms_per_step": ser_ms if ser_ms > 0 else None,
                           "copies": "h2d: the lower triangle of Kbar from pinned host memory in 256-column "
                                     "panels (hf_upload_lower; the upper triangle is never read), step s+1's "
                                     "copy on the library's upload stream during step s (two device K "
                                     "buffers), step 0's not overlapped; d2h: S22, Pi, D and the "
                                     "convergence flag, every step"}
        else:
            line["e2e"] = {"value": None, "unit": "TFLOP/s", "unavailable": e2e_err or "failed on another rank"}

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cb_mode = args.cpu_baseline
    if cb_mode == "auto":
        cb_mode = "full" if spec.L <= 16384 else "sample"
    if rank == 0 and world == 1 and cb_mode != "none" and not args.no_cpu_baseline:
        try:
            Kh_np = Kb.cpu().numpy()
            if cb_mode == "full":
                f, s_, desc = oracle_full(Kh_np, spec)
            else:
                f, s_, desc = oracle_sample(Kh_np, spec, pivots=args.pivots_sample)
            line["cpu_baseline"] = {"value": f / s_ / 1e12, "unit": "TFLOP/s", "cores": host_cores(),
                                    "kind": "oracle", "sample": desc, "seconds": s_}
        except Exception as e:   # the oracle is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": host_cores(), "kind": "oracle",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
