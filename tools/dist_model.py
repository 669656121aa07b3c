"""Per-rank time model of the DISTRIBUTED stage 1 (k_dist.cu) from kernel times
measured on ONE B200 (this run has no multi-GPU box): VERDICT r01 item 2.

  T1  : the one-GPU stage 1 (hf_factor_lowprec, CUDA events) on the config.
  emul: the G-rank emulation on one GPU (hf_set_stage1_partitions(G)): every
        rank's trailing update and panel gather are separate launches timed per
        rank ("trailing@h", "gather@h"), each alone on a full GPU as it would run
        on its own; the chain runs all ranks' CTAs in one cooperative launch with
        the real per-rank geometry (nsm / G CTAs per rank).
  model (serial schedule, what k_dist.cu does):
        T_G = chain_emul + n_pivots * dNV                (NVLink latency per pivot)
            + sum over panels of max-rank trailing       (approximated by max_h sum)
            + max_h gather@h + remote panel bytes / BW   (the panel broadcast)
            + 2 barriers per panel * t_bar + factor-row gather bytes / BW
        dNV = extra latency of the two cross-GPU hops of a pivot (key store into the
        peers' slots; column + mailbox peer read) over their local-L2 versions in the
        emulation: 2 x (1834 - 234) cycles at 1.965 GHz = 1.6 us (peer-LDG vs local L2
        latency, /opt/skills/guides/B300_MICROARCH.md NVLink section); 2.0 us used.
        BW = 770 GB/s peer copy per direction (B200_PROFILING.md); t_bar = 4 us.

    python tools/dist_model.py [config=C4] [G list=2,4,8] > profiles/dist_model_r02.json
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hf_inputs as hi  # noqa: E402
from paper_2208_01907_b200 import hf  # noqa: E402

DNV_US = 2.0
BW = 770e9
T_BAR_US = 4.0


def timed_factor(ctx, K, spec, G):
    if G:
        hf.hf_set_stage1_partitions(ctx, G)
    try:
        ctx.set_profiling(True)
        base = {}
        names = ["chain", "trailing", "other"] + [f"trailing@{h}" for h in range(G or 1)] + \
                [f"gather@{h}" for h in range(G or 1)]
        for c in names:
            base[c] = ctx.kernel_stats(c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = {c: ctx.kernel_stats(c) for c in names}
        ctx.set_profiling(False)
        d = {c: st[c][0] - base[c][0] for c in names}
        nl = {c: st[c][1] - base[c][1] for c in names}
        out = (ms, d, nl, lf.L - lf.n2_tau_only, lf)
    finally:
        if G:
            hf.hf_set_stage1_partitions(ctx, 0)
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
    spec = hi.CONFIGS[name]
    L = spec.L
    K = hi.make_kbar(name, 0, device="cuda")
    ctx = hf.Context(0)
    hf.hf_scale(ctx, K)
    # warm-up (workspace cache), then the one-GPU reference
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
    p1, D1, _ = lf.export(with_L=False)
    lf.close()
    ms1, d1, n1, Ntau, lf = timed_factor(ctx, K, spec, 0)
    lf.close()
    res = {"config": name, "L": L, "one_gpu": {"stage1_ms": ms1, "chain_ms": d1["chain"],
                                              "trailing_ms": d1["trailing"], "other_ms": d1["other"],
                                              "chain_us_per_pivot": d1["chain"] * 1e3 / Ntau},
           "assumptions": {"dNV_us_per_pivot": DNV_US, "peer_GBps": BW / 1e9, "barrier_us": T_BAR_US}, "G": {}}
    for G in Gs:
        ms, d, nl, Ntau_g, lfg = timed_factor(ctx, K, spec, G)
        pg, Dg, _ = lfg.export(with_L=False)
        bitwise = bool((pg == p1).all() and (Dg == D1).all())
        lfg.close()
        npan = int(nl["chain"])
        tr = [d[f"trailing@{h}"] for h in range(G)]
        ga = [d[f"gather@{h}"] for h in range(G)]
        # remote bytes of the panel gathers: every row's s for every pivot, (G-1)/G from peers
        m = torch.arange(L, L - Ntau_g, -1, dtype=torch.float64)
        remote = float(m.sum()) * 4.0 * (G - 1) / G
        Lgather = float(L - spec.n_min) ** 2 * 4.0 * (G - 1) / G
        chain_real = d["chain"] + Ntau_g * DNV_US * 1e-3
        t_model = (chain_real + max(tr) + max(ga) + remote / BW * 1e3 + 2 * npan * T_BAR_US * 1e-3
                   + Lgather / BW * 1e3)
        res["G"][G] = {"bitwise_vs_one_gpu": bitwise, "emul_total_ms": ms, "panels": npan,
                       "chain_emul_ms": d["chain"], "chain_emul_us_per_pivot": d["chain"] * 1e3 / Ntau_g,
                       "chain_real_model_ms": chain_real,
                       "trailing_per_rank_ms": tr, "trailing_imbalance": max(tr) / (sum(tr) / G),
                       "gather_per_rank_ms": ga, "remote_panel_bytes": remote, "factor_gather_bytes": Lgather,
                       "model_ms": t_model, "model_speedup": ms1 / t_model}
        print(json.dumps({G: res["G"][G]}), file=sys.stderr, flush=True)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
