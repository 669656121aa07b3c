"""Host logic of bench.py's work model (no GPU): the algorithmic flop counts that turn the
timed step into TFLOP/s and the rooflines' executed-work figures, checked against brute-force
counts of what the algorithms do."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("L,Ntau", [(7, 7), (40, 33), (300, 299)])
def test_stage1_flops_are_the_rank1_updates_of_the_lower_triangle(L, Ntau):
    """F1 = sum over accepted pivots of 2 x (entries of the remaining lower triangle below the
    pivot): brute force over the steps of P:64-67."""
    brute = 0.0
    for k in range(Ntau):
        m = L - k                        # active size when pivot k is taken
        brute += 2.0 * (m - 1) * m / 2.0  # one FMA per entry of the (m-1) x (m-1) lower triangle
    fm = bench.flop_model(L, Ntau, Ntau, L - Ntau, 3)
    assert fm["stage1"] == pytest.approx(brute, rel=1e-12)


@pytest.mark.parametrize("iters", [1, 2, 6])
def test_gcr_flops_follow_block_gcr(iters):
    """Alg. 5 as gcr.cu runs it: (iters + 2) mat-vecs, (iters + 1) preconditioner applications,
    per iteration the Gram / update products and, on non-final iterations, the
    orthogonalisation against all earlier blocks -- counted step by step here."""
    N, n2 = 1000, 24
    mv = 2.0 * N * N * n2
    count = 2 * mv + 2 * (2.0 * N * N * n2)       # r_0 = b - A x_0, q_0; x_0, p_0 preconditioned
    small = 0.0
    for n in range(iters):
        count += 4 * 2.0 * N * n2 * n2             # M_n, A_n, x += p C, r -= q C
        small += 2.0 * n2 ** 3                     # C = M^-1 A
        if n + 1 < iters:                          # z_{n+1}, w_{n+1}, Q^T z, P / Q updates, G_m
            count += mv + 2.0 * N * N * n2
            count += 3 * (n + 1) * 2.0 * N * n2 * n2
            small += (n + 1) * 2.0 * n2 ** 3
    count += mv                                    # the reported true residual
    fm = bench.flop_model(N + n2, N, N, n2, iters)
    assert fm["gcr"] == pytest.approx(count + small, rel=1e-12)
    assert fm["matvec"] == pytest.approx((iters + 2) * mv, rel=1e-12)
    assert fm["total"] == pytest.approx(fm["stage1"] + fm["gcr"] + fm["schur"] + fm["hard"], rel=1e-12)
    # with the mat-vecs on the int8 tensor cores they leave the DMMA class, nothing else does
    fo = bench.flop_model(N + n2, N, N, n2, iters, ozaki=True)
    assert fm["dmma"] - fo["dmma"] == pytest.approx(fm["matvec"], rel=1e-12)
    assert fo["total"] == fm["total"]


@pytest.mark.parametrize("N,n2", [(100, 8), (5000, 256), (16128, 256)])
def test_blocked_preconditioner_executed_bf16_work(N, n2, monkeypatch):
    """rooflines.trsm's executed bf16 flops = 6 part products x every product the blocked solve
    issues, enumerated block step by block step for both directions (k_trsm_blk.cu)."""
    monkeypatch.delenv("HF_PRECOND", raising=False)
    BS = 64
    while BS < 2048 and BS < N:
        BS *= 2
    nb = -(-N // BS)
    Nb = nb * BS
    ncp = -(-n2 // 8) * 8
    per_dir = 0.0
    for j in range(nb):
        per_dir += 2.0 * BS * BS * ncp                      # the diagonal-block inverse product
        if j + 1 < nb:
            per_dir += 2.0 * BS * BS * ncp                  # the coupling to block j + 1
        if j + 2 < nb:
            per_dir += 2.0 * (Nb - (j + 2) * BS) * BS * ncp  # the bulk update beyond
    iters = 5
    r = bench.trsm_roofline(N, n2, iters, 2.0 * N * N * n2 * (iters + 1), 1.0, 0.5, 1.0, 1.0)
    assert r["bf16_flops_per_step"] == pytest.approx(6 * 2 * per_dir * (iters + 1), rel=1e-12)
    assert r["block_rows"] == BS and r["blocks"] == nb
    if N == 16128:   # C2, 6 applications: x 2 directions x (8 + 7 + 3 x 6) + 2 x 5 + 12
        assert r["library_launches_per_step"] == (iters + 1) * 2 * 33 + 10 + 12


def test_launch_summary_separates_library_kernels(tmp_path):
    """tools/launch_summary.py: libhf's kernels (namespace hf::) per factorization, the library
    kernels apart."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import launch_summary
    rows = ['"ID","API Stream","Block Size","Grid Size","Device","CC","Context","Stream","Kernel Name",'
            '"Section Name","Metric Name","Metric Unit","Metric Value"']
    def row(i, name, ns):
        return f'"{i}","1","(256,1,1)","(1,1,1)","0","10.0","1","7","{name}","Command line profiler metrics",' \
               f'"gpu__time_duration.sum","ns","{ns}"'
    rows += [row(0, "void hf::<unnamed>::k_chain(hf::<unnamed>::ChainArgs)", 4000000),
             row(1, "void hf::<unnamed>::k_chain(hf::<unnamed>::ChainArgs)", 2000000),
             row(2, "nvjet_tss_64x64_64x16_2x2_2cta_h_badd_NNT", 1000000)]
    p = tmp_path / "l.csv"
    p.write_text("\n".join(rows) + "\n")
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        launch_summary.main(str(p), 2)
    out = buf.getvalue()
    line = [l for l in out.splitlines() if l.startswith("k_chain")][0].split()
    assert float(line[1]) == 1.0 and float(line[2]) == pytest.approx(3.0)   # launches, ms per factorization
    assert "library kernels" in out and "nvjet_tss_64x64" in out
    assert np.isclose(float(out.split("launches, ")[1].split(" ms")[0]), 0.5)
