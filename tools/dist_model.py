"""Per-rank time model of the DISTRIBUTED stage 1 (k_dist.cu) from kernel times
measured on ONE B200 (this run has no multi-GPU box): VERDICT r01 item 2.

  T1    the one-GPU stage 1 (hf_factor_lowprec, CUDA events) on the config.
  emul  the G-rank emulation on one GPU (hf_set_stage1_partitions(G),
        HF_DIST_PANEL_TIMES): per panel p the chain's device time (all ranks'
        CTAs in one cooperative launch, the real per-rank geometry) and per rank
        its panel gather and its trailing update (separate launches, each alone
        on a full GPU, as it runs on its own GPU).
  model (per panel p; nbp pivots; every quantity measured unless marked *):
    chain_p*  = chain_emul_p + nbp * dNV + t_bar
    upd_p*    = max_h gather_ph + remote_p / BW + max_h trail_ph + t_bar
    serial    : T = sum_p (chain_p + upd_p)                       (HF_DIST_LOOKAHEAD=0)
    lookahead : T = chain_0 + sum_p max(CONC * chain_{p+1}, upd_p * nsm / (nsm - Cper))
                (the chain of panel p+1 beside panel p's update on the other SMs;
                 chain and update times from the lookahead geometry, measured with
                 HF_DIST_LOOKAHEAD=2: the lookahead kernels on one stream)
    + factor-row gather (N^2 (G-1)/G * 4 bytes / BW) at the end.
  * dNV = extra latency of the two cross-GPU hops of a pivot (key store into the
    peers' slots; column + mailbox peer read) over their local-L2 versions in the
    emulation: 2 x (1834 - 234) cycles / 1.965 GHz = 1.6 us (peer-LDG vs local-L2
    latency, /opt/skills/guides/B300_MICROARCH.md NVLink section); 2.0 us used.
    BW = 770 GB/s peer copy per direction (B200_PROFILING.md); t_bar = 4 us per
    device-side NVLink barrier (one remote atomic + poll); remote_p = m_p nbp 4 B
    (G-1)/G (the panel broadcast).

  full hybrid (Alg. 1 steps 1-5): scale + stage 1 (model above) + stage 2 sharded over the
    right-hand sides (each rank's block GCR + S22 slice timed ALONE on this GPU through
    hf_set_virtual_rank: what it runs on its own GPU) + the S22 / X12 slice broadcast at BW +
    the replicated hard factorization.

    python tools/dist_model.py [config=C4] [G list=2,4,8] > profiles/dist_model_r02.json
"""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DNV_US = 2.0
# the chain runs this much slower beside a concurrent trailing update on the other SMs
# (measured on one B200 at C2 through the same kernels, G = 1 with 64 reserved chain SMs:
# chain 95.8 ms with the lookahead vs 61.1 ms serial, profiles/dist_lookahead_c2_r02.log)
CONC = 95.8 / 61.1
BW = 770e9
T_BAR_US = 4.0
NSM = 148


def worker(name, G, mode):
    """One factorization in this process; stderr of libhf captured through fd 2."""
    import torch
    import hf_inputs as hi
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    K = hi.make_kbar(name, 0, device="cuda")
    torch.cuda.empty_cache()   # the generator's temporaries (C4: 39 GB) back to the device
    ctx = hf.Context(0)
    hf.hf_scale(ctx, K)
    if G:
        hf.hf_set_stage1_partitions(ctx, G)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)   # warm-up (workspace cache)
    lf.close()
    tmp = tempfile.TemporaryFile(mode="w+")
    saved = os.dup(2)
    os.dup2(tmp.fileno(), 2)
    try:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
        e1.record()
        torch.cuda.synchronize()
    finally:
        os.dup2(saved, 2)
        os.close(saved)
    tmp.seek(0)
    panels = None
    for line in tmp.read().splitlines():
        if line.startswith("[hf dist panels] "):
            panels = json.loads(line[len("[hf dist panels] "):])
    perm, D, _ = lf.export(with_L=False)
    out = {"ms": e0.elapsed_time(e1), "Ntau": lf.L - lf.n2_tau_only, "N": lf.N, "panels": panels,
           "perm_hash": hashlib.sha256(perm.tobytes()).hexdigest(), "D_hash": hashlib.sha256(D.tobytes()).hexdigest()}
    print(json.dumps(out), flush=True)


def worker_stage2(name, Gs):
    """Stage 2 (block GCR + S22 slice) of the RHS-sharded multi-GPU path: each rank's own
    slice measured alone on this GPU (hf_set_virtual_rank), ranks 0 and G-1; G = 1 is the
    one-GPU stage 2.  Also the one-GPU scale and hard-factor times."""
    import torch
    import hf_inputs as hi
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    K = hi.make_kbar(name, 0, device="cuda")
    torch.cuda.empty_cache()   # the generator's temporaries (C4: 39 GB) back to the device
    ctx = hf.Context(0)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    hf.hf_scale(ctx, K)
    e[1].record()
    torch.cuda.synchronize()
    scale_ms = e[0].elapsed_time(e[1])
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
    out = {"scale_ms": scale_ms, "n2": lf.n2, "stage2": {}}
    for G in Gs:
        per = []
        for r in ([0, G - 1] if G > 1 else [0]):
            hf.hf_set_virtual_rank(ctx, r, G) if G > 1 else hf.hf_set_virtual_rank(ctx, 0, 0)
            # warm-up run first: the library GEMMs' plans (cuBLASLt heuristics, once per shape
            # and process) and the device cache's first mappings are not per-factorization costs
            hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True)
            hy.close()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True)
            e1.record()
            torch.cuda.synchronize()
            per.append({"rank": r, "iters": info.iters, "true_res": info.max_rel_res_true,
                        "ms": e0.elapsed_time(e1)})
            if G == 1:
                e0.record()
                hf.hf_factor_hard(ctx, hy)
                e1.record()
                torch.cuda.synchronize()
                out["hard_ms"] = e0.elapsed_time(e1)
            hy.close()
        out["stage2"][G] = per
    hf.hf_set_virtual_rank(ctx, 0, 0)
    print(json.dumps(out), flush=True)


def run(name, G, mode):
    env = dict(os.environ, HF_DIST_LOOKAHEAD=str(mode), HF_DIST_PANEL_TIMES="1")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--worker", name, str(G), str(mode)],
                       capture_output=True, text=True, env=env, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def model(res1, resG, L, G, look):
    panels = resG["panels"]
    n = len(panels)
    Ntau = resG["Ntau"]
    nbp_list = []
    left = Ntau
    nbp0 = None
    # panel widths: equal panels of nb except the last (nb recovered from the pivot count)
    nb = -(-Ntau // n) if n else 0
    for p in range(n):
        w = min(nb, left)
        nbp_list.append(w)
        left -= w
    m = L
    ch, up = [], []
    for p, pan in enumerate(panels):
        w = nbp_list[p]
        ch.append(pan["chain"] + w * DNV_US * 1e-3 + T_BAR_US * 1e-3)
        if pan["ranks"]:
            mp = m - w
            remote = mp * w * 4.0 * (G - 1) / G
            up.append(max(r[0] for r in pan["ranks"]) + remote / BW * 1e3 + max(r[1] for r in pan["ranks"])
                      + T_BAR_US * 1e-3)
        else:
            up.append(0.0)
        m -= w
    Lg = float(res1["N"]) ** 2 * 4.0 * (G - 1) / G / BW * 1e3
    if not look:
        T = sum(ch) + sum(up) + Lg
    else:
        cper = max(1, NSM // G)
        s = NSM / (NSM - cper)
        T = ch[0]
        for p in range(n):
            nxt = ch[p + 1] * CONC if p + 1 < n else 0.0
            T += max(nxt, up[p] * s)
        T += Lg
    return {"model_ms": T, "chain_ms_sum": sum(ch), "update_ms_sum": sum(up), "panels": n, "nb": nb,
            "factor_gather_ms": Lg}


def main():
    if sys.argv[1:2] == ["--worker"]:
        return worker(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    if sys.argv[1:2] == ["--stage2"]:
        return worker_stage2(sys.argv[2], [int(x) for x in sys.argv[3].split(",")])
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
    import hf_inputs as hi
    L = hi.CONFIGS[name].L
    one = run(name, 0, 0)
    res = {"config": name, "L": L, "one_gpu_stage1_ms": one["ms"],
           "assumptions": {"dNV_us_per_pivot": DNV_US, "peer_GBps": BW / 1e9, "barrier_us": T_BAR_US,
                           "lookahead_trailing_slowdown": "nsm / (nsm - nsm // G)",
                           "lookahead_chain_slowdown_measured": CONC}, "G": {}}
    for G in Gs:
        rs = run(name, G, 0)
        rl = run(name, G, 2)
        ms_ = model(one, rs, L, G, False)
        ml_ = model(one, rl, L, G, True)
        res["G"][G] = {"bitwise_vs_one_gpu": rs["perm_hash"] == one["perm_hash"] and rs["D_hash"] == one["D_hash"]
                       and rl["perm_hash"] == one["perm_hash"] and rl["D_hash"] == one["D_hash"],
                       "serial": dict(ms_, speedup=one["ms"] / ms_["model_ms"], emul_total_ms=rs["ms"]),
                       "lookahead": dict(ml_, speedup=one["ms"] / ml_["model_ms"], emul_total_ms=rl["ms"])}
        print(json.dumps({G: res["G"][G]}), file=sys.stderr, flush=True)
    # the whole hybrid factorization (Alg. 1 steps 1-5): stage 2 sharded over the right-hand
    # sides (each rank's slice timed alone on this GPU, the slower of ranks 0 and G-1), the
    # S22 / X12 slices broadcast at 770 GB/s, scale and hard factor replicated
    r2 = subprocess.run([sys.executable, os.path.abspath(__file__), "--stage2", name,
                         ",".join(str(g) for g in [1] + Gs)], capture_output=True, text=True, timeout=1800)
    if r2.returncode == 0:
        s2 = json.loads(r2.stdout.strip().splitlines()[-1])
        n2 = s2["n2"]
        t1_full = s2["scale_ms"] + one["ms"] + s2["stage2"]["1"][0]["ms"] + s2.get("hard_ms", 0.0)
        res["full_hybrid"] = {"one_gpu_ms": t1_full, "scale_ms": s2["scale_ms"], "hard_ms": s2.get("hard_ms"),
                              "stage2_one_gpu": s2["stage2"]["1"], "G": {}}
        for G in Gs:
            st2 = max(p["ms"] for p in s2["stage2"][str(G)])
            slices = (n2 * n2 + float(hi.CONFIGS[name].L - n2) * n2) * 8.0 * (G - 1) / G   # S22 + X12 slices
            tG = s2["scale_ms"] + res["G"][G]["serial"]["model_ms"] + st2 + slices / BW * 1e3 + s2.get("hard_ms", 0.0)
            res["full_hybrid"]["G"][G] = {"stage2_per_rank": s2["stage2"][str(G)], "stage2_ms": st2,
                                          "slice_exchange_ms": slices / BW * 1e3, "model_ms": tG,
                                          "speedup": t1_full / tG}
        print(json.dumps({"full_hybrid": res["full_hybrid"]}), file=sys.stderr, flush=True)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
