"""Physics validation of GPU output -- the reference's `hydrobench validate`
suite (proj/src/validation.cpp:25-215) with every time step run by
libhydro_b200.so.

    python -m paper_2106_13465_b200.validation [--flux hllc|exact10] [--math bitwise|tolerance]

prints one PASS/FAIL line per check and "N/M checks passed" like the
reference CLI (tools/hydrobench.cpp:77-88).  The ground truth is a host-side
restatement of the reference's exact Riemann solver
(proj/src/exact_riemann.cpp): Newton on the pressure function to a 1e-14
step, the closed-form two-rarefaction root, bisection as an independent
cross-check, and the self-similar sampler.
"""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass

import numpy as np

from . import hydro as H
from . import slab as S

GAMMA = 1.4


# ---- exact Riemann solver (host) -------------------------------------------

@dataclass
class Waves:
    p_star: float
    u_star: float
    rho_l: float
    rho_r: float
    left_shock: bool
    right_shock: bool
    left_head: float
    left_tail: float
    right_head: float
    right_tail: float
    iterations: int


def _side(w, g):
    return w[0], w[1], w[3], math.sqrt(g * w[3] / w[0])


def _f(p, s, g):
    rho, _, pk, c = s
    if p > pk:
        a = 2.0 / ((g + 1.0) * rho)
        b = (g - 1.0) / (g + 1.0) * pk
        return (p - pk) * math.sqrt(a / (p + b))
    return 2.0 * c / (g - 1.0) * (math.pow(p / pk, (g - 1.0) / (2.0 * g)) - 1.0)


def _df(p, s, g):
    rho, _, pk, c = s
    if p > pk:
        a = 2.0 / ((g + 1.0) * rho)
        b = (g - 1.0) / (g + 1.0) * pk
        root = math.sqrt(a / (p + b))
        return root * (1.0 - 0.5 * (p - pk) / (p + b))
    return 1.0 / (rho * c) * math.pow(p / pk, -(g + 1.0) / (2.0 * g))


def exact_riemann(wl, wr, g=GAMMA) -> Waves:
    """exact_riemann (exact_riemann.cpp:136-202) on primitive states
    (rho, u, v, p)."""
    l, r = _side(wl, g), _side(wr, g)
    du = wr[1] - wl[1]
    if 2.0 * (l[3] + r[3]) / (g - 1.0) <= du:
        raise H.HydroError(H.ErrorCategory.VALIDATION,
                           "vacuum-generating Riemann states are out of scope")
    p_min = min(l[2], r[2])
    iters = 0
    if _f(p_min, l, g) + _f(p_min, r, g) + du >= 0.0:
        z = (g - 1.0) / (2.0 * g)
        num = l[3] + r[3] - 0.5 * (g - 1.0) * du
        den = l[3] / math.pow(l[2], z) + r[3] / math.pow(r[2], z)
        p = math.pow(num / den, 1.0 / z)
    else:
        p = max(0.5 * (l[2] + r[2]) - 0.125 * du * (l[0] + r[0]) * (l[3] + r[3]), p_min)
        while iters < 100:
            f = _f(p, l, g) + _f(p, r, g) + du
            nxt = p - f / (_df(p, l, g) + _df(p, r, g))
            nxt = max(nxt, p_min)
            change = abs(nxt - p)
            p = nxt
            iters += 1
            if change <= 1e-14 * p:
                break
    u = 0.5 * (wl[1] + wr[1]) + 0.5 * (_f(p, r, g) - _f(p, l, g))
    gm = (g - 1.0) / (g + 1.0)

    def star(s, sign):
        rho, uk, pk, c = s
        if p > pk:
            ratio = p / pk
            head = uk + sign * c * math.sqrt((g + 1.0) / (2.0 * g) * ratio + (g - 1.0) / (2.0 * g))
            return True, head, head, rho * (ratio + gm) / (gm * ratio + 1.0)
        c_star = c * math.pow(p / pk, (g - 1.0) / (2.0 * g))
        return False, uk + sign * c, u + sign * c_star, rho * math.pow(p / pk, 1.0 / g)

    ls, lh, lt, rl = star(l, -1.0)
    rs, rh, rt, rr = star(r, +1.0)
    return Waves(p, u, rl, rr, ls, rs, lh, lt, rh, rt, iters)


def pstar_bisect(wl, wr, g=GAMMA) -> float:
    """riemann_pstar_bisect (exact_riemann.cpp:99-134)."""
    l, r = _side(wl, g), _side(wr, g)
    du = wr[1] - wl[1]
    fn = lambda p: _f(p, l, g) + _f(p, r, g) + du  # noqa: E731
    lo, hi = min(l[2], r[2]), max(l[2], r[2])
    if fn(lo) >= 0.0:
        hi = lo
        while fn(lo) >= 0.0:
            lo *= 0.5
    else:
        while fn(hi) < 0.0:
            hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if fn(mid) < 0.0:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-14 * hi:
            break
    return 0.5 * (lo + hi)


def sample(ws: Waves, wl, wr, xi, g=GAMMA):
    """sample_riemann (exact_riemann.cpp:204-241) -> (rho, u, v, p)."""
    if xi <= ws.u_star:
        rho, uk, pk, c = _side(wl, g)
        if xi <= ws.left_head:
            return tuple(wl)
        if ws.left_shock or xi >= ws.left_tail:
            return ws.rho_l, ws.u_star, wl[2], ws.p_star
        u = 2.0 / (g + 1.0) * (c + 0.5 * (g - 1.0) * uk + xi)
        cc = 2.0 / (g + 1.0) * (c + 0.5 * (g - 1.0) * (uk - xi))
        return (rho * math.pow(cc / c, 2.0 / (g - 1.0)), u, wl[2],
                pk * math.pow(cc / c, 2.0 * g / (g - 1.0)))
    rho, uk, pk, c = _side(wr, g)
    if xi >= ws.right_head:
        return tuple(wr)
    if ws.right_shock or xi <= ws.right_tail:
        return ws.rho_r, ws.u_star, wr[2], ws.p_star
    u = 2.0 / (g + 1.0) * (-c + 0.5 * (g - 1.0) * uk + xi)
    cc = 2.0 / (g + 1.0) * (c - 0.5 * (g - 1.0) * (uk - xi))
    return (rho * math.pow(cc / c, 2.0 / (g - 1.0)), u, wr[2],
            pk * math.pow(cc / c, 2.0 * g / (g - 1.0)))


# ---- checks ------------------------------------------------------------------

@dataclass
class CheckResult:
    name: str
    passed: bool
    detail: str


def check_riemann_solver() -> list[CheckResult]:
    """validation.cpp:25-103 on the host solver used as ground truth below."""
    out = []
    w = (1.0, 0.0, 0.0, 1.0)
    ws = exact_riemann(w, w)
    pe, ue = abs(ws.p_star - 1.0), abs(ws.u_star)
    out.append(CheckResult("riemann-static", pe <= 1e-12 and ue <= 1e-12,
                           f"|p*-p|={pe:.3g} |u*|={ue:.3g} (tol 1e-12)"))
    ws = exact_riemann((1.0, 0.0, 0.0, 1.0), (0.125, 0.0, 0.0, 0.1))
    ok = (abs(ws.p_star - 0.30313) <= 5e-6 and abs(ws.u_star - 0.92745) <= 5e-6
          and not ws.left_shock and ws.right_shock)
    out.append(CheckResult("riemann-sod", ok, f"p*={ws.p_star:.7f} u*={ws.u_star:.7f} "
                           "(expected 0.30313 / 0.92745 to 5e-6)"))
    ws = exact_riemann((1.0, 2.0, 0.0, 1.0), (1.0, -2.0, 0.0, 1.0))
    out.append(CheckResult("riemann-symmetric", abs(ws.u_star) <= 1e-14,
                           f"|u*|={abs(ws.u_star):.3g} (tol 1e-14)"))
    rng = np.random.default_rng(20240811)
    worst, tested = 0.0, 0
    while tested < 2000:
        wl = (10 ** rng.uniform(-2, 2), rng.uniform(-3, 3), 0.0, 10 ** rng.uniform(-2, 2))
        wr = (10 ** rng.uniform(-2, 2), rng.uniform(-3, 3), 0.0, 10 ** rng.uniform(-2, 2))
        cl, cr = math.sqrt(GAMMA * wl[3] / wl[0]), math.sqrt(GAMMA * wr[3] / wr[0])
        if 0.8 * 2.0 * (cl + cr) / (GAMMA - 1.0) <= wr[1] - wl[1]:
            continue
        a, b = exact_riemann(wl, wr).p_star, pstar_bisect(wl, wr)
        worst = max(worst, abs(a - b) / max(a, b))
        tested += 1
    out.append(CheckResult("riemann-rootfinder-agreement", worst <= 1e-12,
                           f"worst relative p* gap {worst:.3g} over {tested} pairs (tol 1e-12)"))
    return out


def _tag(flux: str, math: str) -> str:
    return ("" if flux == "hllc" else "-" + flux) + ("" if math == "bitwise" else "-" + math)


def check_sod_profile(flux: str = "hllc", math: str = "bitwise") -> CheckResult:
    """validation.cpp:105-139: the 4-row Sod tube to t=0.2 on the GPU."""
    model = H.GasModel()
    n = 200
    grid = H.make_case("sod", 4, n, model)
    H.run_until_gpu(grid, model, 0.2, "reflect", flux=flux, math=math)
    inner = grid.interior()
    transverse = float(np.max(np.abs(inner[:, 1:, :] - inner[:, :1, :])))
    ws = exact_riemann((1.0, 0.0, 0.0, 1.0), (0.125, 0.0, 0.0, 0.1))
    dy = 1.0 / n
    l1 = 0.0
    for j in range(1, n + 1):
        xi = ((j - 0.5) * dy - 0.5) / 0.2
        l1 += abs(inner[0, 0, j - 1] - sample(ws, (1.0, 0.0, 0.0, 1.0), (0.125, 0.0, 0.0, 0.1), xi)[0]) * dy
    return CheckResult(f"sod-density-l1{_tag(flux, math)}",
                       transverse <= 1e-13 and l1 < 1e-2,
                       f"L1={l1:.5f} (tol 1e-2), transverse spread {transverse:.3g} (tol 1e-13)")


def _pairwise(v: np.ndarray) -> float:
    """pairwise_sum (audit.cpp:16-25): halve until blocks of <= 8."""
    if v.size <= 8:
        s = 0.0
        for x in v:
            s += float(x)
        return s
    h = v.size // 2
    return _pairwise(v[:h]) + _pairwise(v[h:])


def _totals(grid: H.Grid2D):
    vol = grid.dx * grid.dy
    return [vol * _pairwise(grid.interior()[v].ravel()) for v in range(4)]


def _asymmetry(grid: H.Grid2D) -> float:
    """mirror_asymmetry (audit.cpp:156-180)."""
    u = grid.interior()
    mx = u[:, ::-1, :].copy()
    mx[1] = -mx[1]
    my = u[:, :, ::-1].copy()
    my[2] = -my[2]
    worst = 0.0
    for m in (mx, my):
        scale = np.maximum(np.maximum(np.abs(u), np.abs(m)), 1.0)
        worst = max(worst, float(np.max(np.abs(u - m) / scale)))
    return worst


def check_conservation(flux: str = "hllc", math: str = "bitwise") -> list[CheckResult]:
    """validation.cpp:141-172: blast, 10 blocks of 10 GPU steps."""
    model = H.GasModel()
    grid = H.make_case("blast", 64, 64, model)
    start = _totals(grid)
    mass = energy = 0.0
    asym = _asymmetry(grid)
    with H.GpuGrid(64, 64, grid.dx, grid.dy, model, "reflect", flux=flux, math=math) as g:
        g.upload(grid.planes)
        for _ in range(10):
            g.run(10)
            g.download(grid.planes)
            now = _totals(grid)
            mass = max(mass, abs(now[0] - start[0]) / abs(start[0]))
            energy = max(energy, abs(now[3] - start[3]) / abs(start[3]))
            asym = max(asym, _asymmetry(grid))
    tag = _tag(flux, math)
    return [CheckResult("conservation-mass" + tag, mass <= 1e-11,
                        f"relative drift {mass:.3g} over 100 steps (tol 1e-11)"),
            CheckResult("conservation-energy" + tag, energy <= 1e-11,
                        f"relative drift {energy:.3g} over 100 steps (tol 1e-11)"),
            CheckResult("blast-mirror-symmetry" + tag, asym <= 1e-12,
                        f"worst per-cell asymmetry {asym:.3g} audited every 10 steps (tol 1e-12)")]


def _first_diff(a: np.ndarray, b: np.ndarray) -> str:
    bad = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
    if not len(bad):
        return "grids bitwise equal"
    v, i, j = bad[0]
    return f"first difference at plane {v} ({i - 1},{j - 1})"


def check_execution_equivalence(math: str = "bitwise") -> list[CheckResult]:
    """The GPU analogue of validation.cpp:174-207: every execution variant of
    the GPU path (work-item segmentation, CUDA-graph replay vs single launches,
    row-slab decomposition with halo swaps) must give the same bits."""
    model = H.GasModel()
    steps = 10
    base = H.make_case("blast", 64, 64, model)
    ref = base.copy()
    with H.GpuGrid(64, 64, ref.dx, ref.dy, model, math=math) as g:
        g.upload(ref.planes)
        g.run(steps)
        g.download(ref.planes)
    out = []
    for seg in ((16, 16), (5, 8), (64, 64)):
        grid = base.copy()
        with H.GpuGrid(64, 64, grid.dx, grid.dy, model, math=math) as g:
            g.tune(seg[0], seg[1], 0)
            g.upload(grid.planes)
            g.run(steps)
            g.download(grid.planes)
        out.append(CheckResult(f"equivalence-segments-{seg[0]}x{seg[1]}{_tag('hllc', math)}",
                               np.array_equal(grid.planes, ref.planes),
                               _first_diff(grid.planes, ref.planes)))
    grid = base.copy()
    with H.GpuGrid(64, 64, grid.dx, grid.dy, model, math=math) as g:
        g.upload(grid.planes)
        for _ in range(steps):  # single steps: no graph, one prologue per call
            g.run(1)
        g.download(grid.planes)
    out.append(CheckResult("equivalence-stepwise" + _tag("hllc", math),
                           np.array_equal(grid.interior(), ref.interior()),
                           _first_diff(grid.interior(), ref.interior())))
    import torch
    for world, p2p in ((2, False), (4, False), (4, True)):
        slabs = []
        for r in range(world):
            sl = S.GpuSlab(S.SlabGeometry(64, 64, r, world), base.dx, base.dy, model, "reflect", 0,
                           math=math)
            sl.bind_stream(torch.cuda.current_stream())
            sl.grid.upload(S.slab_planes(base.planes, 64, world, r))
            slabs.append(sl)
        S.run_loopback(slabs, steps, p2p=p2p)
        torch.cuda.synchronize()
        parts = []
        for sl in slabs:
            p = np.zeros((4, sl.geo.nx + 4, 68))
            sl.grid.download(p)
            parts.append(p)
        got = S.gather_planes(parts, 64, 64)
        name = f"equivalence-slabs-{world}" + ("-peer-halo" if p2p else "") + _tag("hllc", math)
        out.append(CheckResult(name, np.array_equal(got, ref.planes), _first_diff(got, ref.planes)))
    return out


def run_validation_suite(flux: str = "hllc", math: str = "bitwise") -> list[CheckResult]:
    results = check_riemann_solver()
    results.append(check_sod_profile(flux, math))
    results += check_conservation(flux, math)
    results += check_execution_equivalence(math)
    return results


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--flux", default="hllc", choices=sorted(H.FLUX))
    ap.add_argument("--math", default="bitwise", choices=sorted(H.MATH))
    args = ap.parse_args(argv)
    results = run_validation_suite(args.flux, args.math)
    failed = 0
    for r in results:
        print(f"{'PASS' if r.passed else 'FAIL'} {r.name}: {r.detail}")
        failed += not r.passed
    print(f"{len(results) - failed}/{len(results)} checks passed")
    return 0 if failed == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
