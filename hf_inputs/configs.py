"""Seeded synthetic inputs with the shapes and structure of BASELINE.json's
configs.  No method arithmetic lives here: the outputs
are the UNSCALED symmetric matrix Kbar (float64) and right-hand sides.

A symmetric matrix has the same bytes in row- and column-major order, so the
torch tensors returned here can be handed to column-major code unchanged.

RNG: torch.Generator seeded with config_seed(name, seed).  Planted matrices
are drawn on the requested device (CPU generator = mt19937, CUDA generator =
Philox-4x32-10); the two devices therefore give DIFFERENT matrices for the
same seed.  Tests and the bench always build a given case on one device and
hand the same bytes to both the oracle and the CUDA path.  The structured
configs (C1, C3) draw only a few numbers with numpy's Philox generator and
are identical on every device.
"""
from __future__ import annotations

import math
import zlib
from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    kind: str                 # planted | neumann | saddle
    L: int
    tau: float = 1e-2
    n_min: int = 0            # postponement floor (reading [R5])
    n_hard: int = 0           # planted: number of hard directions
    u_hard: tuple = (0.0, 0.0)
    u_rest: tuple = (-2.0, 0.0)
    p_neg: float = 0.3
    grid: int = 0             # neumann / saddle: nodes per side
    n_incl: int = 0           # neumann: inclusions
    incl_size: int = 0        # neumann: inclusion side (nodes)
    jump: float = 1.0         # saddle: coefficient jump across the line
    k_in: float = 1e6         # neumann: coefficient inside inclusions
    k_link: float = 1e-8      # neumann: coefficient of the edges joining them to the bulk
    delta: float = 0.0        # stokes_ns: stabilisation weight of the pressure block


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C0": ConfigSpec("C0", "planted", 256, n_min=4, n_hard=4, u_hard=(-10.0, -8.0)),
    "C1": ConfigSpec("C1", "neumann", 64 * 64, grid=64, n_incl=3, incl_size=8),
    # n_min: 64 planted directions, but at L = 16384 the FP32 factor leaves more unresolved
    # directions (Gaussian B, bulk condition ~ 4 L^2 100); DESIGN.md [R5]
    "C2": ConfigSpec("C2", "planted", 16384, n_min=256, n_hard=64, u_hard=(-12.0, -6.0)),
    "C3": ConfigSpec("C3", "saddle", 2 * 96 * 96 + 2 * 48 * 48, grid=96, jump=1e4),
    # n_min: 256 planted directions; with n_min = 256 block GCR stagnates at 3e-6 after 100
    # iterations, 512 converges in 20 (DESIGN.md [R5])
    "C4": ConfigSpec("C4", "planted", 65536, n_min=512, n_hard=256, u_hard=(-12.0, -6.0)),
    # small analogs with the same recipes (tests; the oracle finishes in seconds)
    "P64": ConfigSpec("P64", "planted", 64, n_min=2, n_hard=2, u_hard=(-10.0, -8.0)),
    "P512": ConfigSpec("P512", "planted", 512, n_min=8, n_hard=8, u_hard=(-12.0, -6.0)),
    "P1024": ConfigSpec("P1024", "planted", 1024, n_min=16, n_hard=16, u_hard=(-12.0, -6.0)),
    "P2048": ConfigSpec("P2048", "planted", 2048, n_min=32, n_hard=32, u_hard=(-12.0, -6.0)),
    "P4096": ConfigSpec("P4096", "planted", 4096, n_min=64, n_hard=64, u_hard=(-12.0, -6.0)),
    "N16": ConfigSpec("N16", "neumann", 16 * 16, grid=16, n_incl=2, incl_size=4),
    "N32": ConfigSpec("N32", "neumann", 32 * 32, grid=32, n_incl=3, incl_size=4),
    "S12": ConfigSpec("S12", "saddle", 2 * 12 * 12 + 2 * 6 * 6, grid=12, jump=1e4),
    "S24": ConfigSpec("S24", "saddle", 2 * 24 * 24 + 2 * 12 * 12, grid=24, jump=1e4),
    # NEXT-3: nonsymmetric [A B^T; -B delta D] (stokes-like) and [A B^T; -B 0] (dd-hole-like)
    "T8": ConfigSpec("T8", "stokes_ns", 2 * 8 * 8 + 2 * 4 * 4, grid=8, jump=1e4, delta=1e-2),
    "H8": ConfigSpec("H8", "stokes_ns", 2 * 8 * 8 + 2 * 4 * 4, grid=8, jump=1e4, delta=0.0),
    "T24": ConfigSpec("T24", "stokes_ns", 2 * 24 * 24 + 2 * 12 * 12, grid=24, jump=1e4, delta=1e-2),
    "T96": ConfigSpec("T96", "stokes_ns", 2 * 96 * 96 + 2 * 48 * 48, grid=96, jump=1e4, delta=1e-2),
}


def config_seed(name: str, seed: int) -> int:
    return (zlib.crc32(name.encode()) * 1_000_003 + int(seed)) % (2**62)


def _spec(cfg) -> ConfigSpec:
    return CONFIGS[cfg] if isinstance(cfg, str) else cfg


# ----------------------------------------------------------------------------
def planted(spec: ConfigSpec, seed: int, device="cpu", chunk_rows: int = 8192) -> torch.Tensor:
    """Kbar = B diag(lambda) B^T, B i.i.d. N(0,1) L x L, lambda_i = +-10^u_i
    (negative with probability p_neg), the first n_hard with u ~ U[u_hard],
    the rest u ~ U[u_rest]; symmetrised from its lower triangle."""
    L = spec.L
    g = torch.Generator(device=device)
    g.manual_seed(config_seed(spec.name, seed))
    B = torch.randn(L, L, generator=g, device=device, dtype=torch.float64)
    u = torch.empty(L, device=device, dtype=torch.float64).uniform_(*spec.u_rest, generator=g)
    if spec.n_hard:
        u[: spec.n_hard].uniform_(*spec.u_hard, generator=g)
    neg = torch.rand(L, generator=g, device=device, dtype=torch.float64) < spec.p_neg
    lam = torch.pow(10.0, u) * torch.where(neg, -1.0, 1.0).to(torch.float64)
    K = torch.empty(L, L, device=device, dtype=torch.float64)
    for r0 in range(0, L, chunk_rows):
        r1 = min(L, r0 + chunk_rows)
        torch.matmul(B[r0:r1] * lam, B.T, out=K[r0:r1])
    del B
    _symmetrize_from_lower(K)
    return K


def _symmetrize_from_lower(K: torch.Tensor, blk: int = 4096) -> None:
    """K[i, j] := K[j, i] for i < j (row-major view: copy the lower triangle
    of the row-major array into its upper triangle) -- in blocks, in place."""
    L = K.shape[0]
    for c0 in range(0, L, blk):
        c1 = min(L, c0 + blk)
        # rows r >= c1 in columns [c0,c1) are strictly lower: mirror them
        if c1 < L:
            K[c0:c1, c1:] = K[c1:, c0:c1].T
        d = K[c0:c1, c0:c1]
        d.copy_(torch.tril(d) + torch.tril(d, -1).T)


def _inclusions(spec: ConfigSpec, seed: int):
    n, s = spec.grid, spec.incl_size
    rng = np.random.Generator(np.random.Philox(config_seed(spec.name + "/incl", seed)))
    boxes = []
    tries = 0
    while len(boxes) < spec.n_incl:
        tries += 1
        if tries > 100000:
            raise RuntimeError("inclusion placement failed")
        x0 = int(rng.integers(1, n - 1 - s + 1))    # nodes x0..x0+s-1 inside 1..n-2
        y0 = int(rng.integers(1, n - 1 - s + 1))
        ok = all(abs(x0 - bx) >= s + 1 or abs(y0 - by) >= s + 1 for bx, by in boxes)
        if ok:
            boxes.append((x0, y0))
    return boxes


def neumann_inclusions(spec: ConfigSpec, seed: int, device="cpu") -> torch.Tensor:
    """Weighted graph Laplacian of the grid x grid 5-point stencil, pure Neumann
    (no Dirichlet rows): edge weight k_in inside one inclusion, k_link when the
    ends are in different inclusions or one end is in the bulk, 1 otherwise."""
    n = spec.grid
    L = n * n
    incl = -np.ones((n, n), dtype=np.int64)          # [y, x]
    for b, (x0, y0) in enumerate(_inclusions(spec, seed)):
        incl[y0:y0 + spec.incl_size, x0:x0 + spec.incl_size] = b
    K = np.zeros((L, L), dtype=np.float64)

    def add(a, b, w):
        K[a, a] += w
        K[b, b] += w
        K[a, b] -= w
        K[b, a] -= w

    for y in range(n):
        for x in range(n):
            a = y * n + x
            for (xx, yy) in ((x + 1, y), (x, y + 1)):
                if xx < n and yy < n:
                    ia, ib = incl[y, x], incl[yy, xx]
                    if ia >= 0 and ia == ib:
                        w = spec.k_in
                    elif ia != ib:
                        w = spec.k_link
                    else:
                        w = 1.0
                    add(a, yy * n + xx, w)
    return torch.from_numpy(K).to(device)


def saddle_point(spec: ConfigSpec, seed: int, device="cpu") -> torch.Tensor:
    """[A B^T; B 0]: A = 2-dof (u_x, u_y interleaved per node, nodes row-major)
    5-point Laplacian on grid x grid nodes, h = 1/(grid-1), edge weight
    (jump or 1)/h^2 by the side of a seeded random line the edge midpoint lies
    on; B: TWO rows per 2x2 macro-cell with lower-left node (x, y) = (2I, 2J),
    the divergence-like differences at its two diagonal corners,
        (u_x(x+1,y)   - u_x(x,y)   + u_y(x,y+1)   - u_y(x,y))   / h
        (u_x(x+1,y+1) - u_x(x,y+1) + u_y(x+1,y+1) - u_y(x+1,y)) / h,
    each with 4 nonzeros +-1/h, so B has 2 (grid/2)^2 rows: 4608 x 18432 at
    grid = 96 and L = 23040 as BASELINE.json's config 3 states.  Pure Neumann."""
    n = spec.grid
    h = 1.0 / (n - 1)
    nv = 2 * n * n
    npc = 2 * (n // 2) ** 2
    L = nv + npc
    assert L == spec.L
    rng = np.random.Generator(np.random.Philox(config_seed(spec.name + "/line", seed)))
    th = float(rng.uniform(0.0, 2.0 * math.pi))
    cx, cy = float(rng.uniform(0.2, 0.8)), float(rng.uniform(0.2, 0.8))
    nx, ny = math.cos(th), math.sin(th)
    K = np.zeros((L, L), dtype=np.float64)

    def node(x, y):
        return y * n + x

    for y in range(n):
        for x in range(n):
            for (xx, yy) in ((x + 1, y), (x, y + 1)):
                if xx < n and yy < n:
                    mx, my = 0.5 * (x + xx) * h, 0.5 * (y + yy) * h
                    w = (spec.jump if (mx - cx) * nx + (my - cy) * ny > 0 else 1.0) / h**2
                    for c in range(2):
                        a, b = 2 * node(x, y) + c, 2 * node(xx, yy) + c
                        K[a, a] += w
                        K[b, b] += w
                        K[a, b] -= w
                        K[b, a] -= w
    for J in range(n // 2):
        for I in range(n // 2):
            x, y = 2 * I, 2 * J
            r = nv + 2 * (J * (n // 2) + I)
            rows = (((2 * node(x + 1, y) + 0, 1.0 / h), (2 * node(x, y) + 0, -1.0 / h),
                     (2 * node(x, y + 1) + 1, 1.0 / h), (2 * node(x, y) + 1, -1.0 / h)),
                    ((2 * node(x + 1, y + 1) + 0, 1.0 / h), (2 * node(x, y + 1) + 0, -1.0 / h),
                     (2 * node(x + 1, y + 1) + 1, 1.0 / h), (2 * node(x + 1, y) + 1, -1.0 / h)))
            for q, row in enumerate(rows):
                for dof, val in row:
                    K[r + q, dof] += val
                    K[dof, r + q] += val
    return torch.from_numpy(K).to(device)


def stokes_ns(spec: ConfigSpec, seed: int, device="cpu") -> torch.Tensor:
    """NONSYMMETRIC [A B^T; -B delta D] (the paper's stokes / dd-hole block
    structure; delta = 0 gives [A B^T; -B 0]):
    A and B exactly as saddle_point on the same grid and seeded line, the
    lower-left block negated, D the graph Laplacian of the pressure unknowns
    (the two unknowns of a macro-cell and the 4-neighbour macro-cells joined
    with weight 1).  Returned as a row-major tensor holding the MATRIX Kbar
    (entry [i, j]); column-major code needs Kbar.T.contiguous() (see colmajor)."""
    n = spec.grid
    base = saddle_point(ConfigSpec(spec.name, "saddle", spec.L, grid=n, jump=spec.jump), seed, "cpu").numpy()
    nv = 2 * n * n
    K = base.copy()
    K[nv:, :nv] *= -1.0
    if spec.delta != 0.0:
        m = n // 2
        D = np.zeros((2 * m * m, 2 * m * m))

        def link(a, b):
            D[a, a] += 1.0
            D[b, b] += 1.0
            D[a, b] -= 1.0
            D[b, a] -= 1.0

        for J in range(m):
            for I in range(m):
                c = 2 * (J * m + I)
                link(c, c + 1)
                if I + 1 < m:
                    link(c, c + 2)
                    link(c + 1, c + 3)
                if J + 1 < m:
                    link(c, c + 2 * m)
                    link(c + 1, c + 2 * m + 1)
        K[nv:, nv:] += spec.delta * D
    return torch.from_numpy(K).to(device)


def colmajor(K: torch.Tensor) -> torch.Tensor:
    """The same matrix laid out column-major (what libhf reads) in a contiguous tensor."""
    return K.T.contiguous()


def make_kbar(cfg, seed: int = 0, device="cpu") -> torch.Tensor:
    spec = _spec(cfg)
    if spec.kind == "planted":
        return planted(spec, seed, device)
    if spec.kind == "neumann":
        return neumann_inclusions(spec, seed, device)
    if spec.kind == "saddle":
        return saddle_point(spec, seed, device)
    if spec.kind == "stokes_ns":
        return stokes_ns(spec, seed, device)
    raise ValueError(spec.kind)


def manufactured_x(L: int, device="cpu") -> torch.Tensor:
    """x*_i = i mod 11 (the paper's manufactured solution)."""
    return (torch.arange(L, device=device, dtype=torch.int64) % 11).to(torch.float64)


def make_rhs(cfg, seed: int = 0, device="cpu") -> torch.Tensor:
    """The config's random right-hand side for the UNSCALED system:
    planted: N(0,1); neumann: N(0,1) minus its mean (consistent with the
    constant kernel); saddle: N(0,1) on the velocity rows, 0 on pressure rows."""
    spec = _spec(cfg)
    g = torch.Generator(device="cpu")
    g.manual_seed(config_seed(spec.name + "/rhs", seed))
    b = torch.randn(spec.L, generator=g, dtype=torch.float64)
    if spec.kind == "neumann":
        b = b - b.mean()
    elif spec.kind == "saddle":
        nv = 2 * spec.grid * spec.grid
        b[nv:] = 0.0
        for c in range(2):
            b[c:nv:2] -= b[c:nv:2].mean()
    return b.to(device)
