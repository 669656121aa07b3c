import sys; sys.path.insert(0, ".")
from fractions import Fraction
import numpy as np, torch
import hf_inputs as hi
from hf_inputs.configs import ConfigSpec
from oracle import exact
from paper_2208_01907_b200 import hf
ctx = hf.Context(0)
spec = ConfigSpec("P48", "planted", 48, n_min=3, n_hard=3, u_hard=(-10.0, -8.0))
K = hi.make_kbar(spec, 0).to("cuda"); hf.hf_scale(ctx, K)
lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=64)
hy, info, S = hf.hf_schur_gcr_dd(ctx, K, lf, want_S22_host=True)
print("schur info", info)
kd = hf.hf_factor_hard(ctx, hy, eps_ker=1e-20); print("kd", kd, hy.hard_export())
Kh = K.cpu().numpy(); L = Kh.shape[0]
perm, _, _ = lf.export64(); lam1, lam2 = list(perm[:lf.N]), list(perm[lf.N:])
b = Kh @ (np.arange(L) % 11.0)
xh, xl, sinfo = hf.hf_solve_dd(ctx, hy, torch.from_numpy(b).cuda()); print("solve info", sinfo)
xh, xl = xh.cpu().numpy(), xl.cpu().numpy()
F = exact.to_fractions(Kh)
x = [Fraction(float(xh[i])) + Fraction(float(xl[i])) for i in range(L)]
r = [Fraction(float(b[i])) - sum(F[i][j] * x[j] for j in range(L)) for i in range(L)]
print("res lam1", float(max(abs(r[i]) for i in lam1)), "res lam2", float(max(abs(r[i]) for i in lam2)), "bmax", np.abs(b).max())
# exact y1 for b1 and compare x on lam2 with exact solution
xe = exact.solve(F, [[Fraction(float(v))] for v in b]); xe = [v[0] for v in xe]
print("err lam1", float(max(abs(x[i]-xe[i]) for i in lam1)), "err lam2", float(max(abs(x[i]-xe[i]) for i in lam2)))
Sh, Sl = S
Sx = exact.schur(Kh, [int(i) for i in lam1], [int(i) for i in lam2])
print("S22 rel err", exact.rel_err(Sx, Sh, Sl))
