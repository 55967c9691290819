"""CPU oracle for the PFASST x multigrid hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``pintlab``
(``/root/reference/pkg/src/pintlab``) for exactly the functions on the hot
path.  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product (``paper_1407_6486_b200``) never imports, links or executes it.

Every function names the reference ``file:line`` it restates.  Element-wise
expressions keep the reference's evaluation order term by term (numpy rounds
after every operation and never contracts to FMA), and the dense
contractions go through ``np.tensordot`` exactly as the reference does, so
on one machine this oracle is bit-identical to the reference.  That claim
is *pinned*, not assumed: ``tests/test_oracle_golden.py`` compares it
bit-for-bit against ``tests/golden/*.npz`` written by ``oracle/make_golden.py``,
which imports and runs the real reference in the build container.

Scope: HeatOperator.apply/diagonal, the transfers,
the Jacobi / jor-rb / lexicographic Gauss-Seidel smoothers, v_cycle and the
FixedCycles / ToTolerance / Direct policies, sdc_sweep, residual, run_sdc,
the FAS machinery, mlsdc_iteration, burn_in, interpolate_up, run_mlsdc and
the serial PFASST schedule.  Out of scope: analysis.py, config.py, cli.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

# ---------------------------------------------------------------------------
# quadrature  (quadrature.py:18-190)


def uniform_nodes(m):
    """quadrature.py:46-50 -- t_i = i/m as exact rationals."""
    if m < 1:
        raise ValueError("need at least one sub-step")
    return tuple(Fraction(i, m) for i in range(m + 1))


def _lagrange(points):
    """Coefficient lists (ascending powers) of the Lagrange cardinal
    polynomials on ``points`` (quadrature.py:71-81)."""
    out = []
    for i, xi in enumerate(points):
        coeffs = [Fraction(1)]
        for j, xj in enumerate(points):
            if i == j:
                continue
            a, b = -xj / (xi - xj), Fraction(1) / (xi - xj)
            nxt = [Fraction(0)] * (len(coeffs) + 1)
            for k, c in enumerate(coeffs):
                nxt[k] += c * a
                nxt[k + 1] += c * b
            coeffs = nxt
        out.append(coeffs)
    return out


def _eval(coeffs, t):
    acc, power = Fraction(0), Fraction(1)
    for c in coeffs:
        acc += c * power
        power *= t
    return acc


@dataclass(frozen=True)
class Table:
    """Q (right-M-node weights) and the sub-step fractions (quadrature.py:84-115)."""
    nodes: tuple
    q: np.ndarray

    @property
    def m(self):
        return len(self.nodes) - 1

    @property
    def gammas(self):
        return tuple(b - a for a, b in zip(self.nodes, self.nodes[1:]))


def make_table(nodes):
    """quadrature.py:102-115: q[row, i] = int_0^{t_row} l_{i}(t) dt over the
    right M nodes, rounded once from the exact rational."""
    m = len(nodes) - 1
    basis = _lagrange(list(nodes[1:]))
    q = np.zeros((m + 1, m + 1))
    for row in range(1, m + 1):
        upper = nodes[row]
        for i in range(1, m + 1):
            total, power = Fraction(0), upper
            for j, c in enumerate(basis[i - 1]):
                total += c * power / (j + 1)
                power *= upper
            q[row, i] = float(total)
    return Table(tuple(nodes), q)


def uniform_table(m):
    """quadrature.py:118-120."""
    return make_table(uniform_nodes(m))


def time_indices(fine_nodes, coarse_nodes):
    """Fine node index of every coarse node (quadrature.py:123-142 +
    hierarchy.py:80-82)."""
    try:
        return [list(fine_nodes).index(t) for t in coarse_nodes]
    except ValueError:
        raise ValueError("node sets are not nested") from None


def correction_interp(coarse_nodes, fine_nodes):
    """quadrature.py:165-190: row 0 selects coarse node 0; other rows
    interpolate on the coarse *quadrature* nodes only."""
    time_indices(fine_nodes, coarse_nodes)
    basis = _lagrange(list(coarse_nodes[1:]))
    p = np.zeros((len(fine_nodes), len(coarse_nodes)))
    p[0, 0] = 1.0
    for row in range(1, len(fine_nodes)):
        for col, poly in enumerate(basis):
            p[row, col + 1] = float(_eval(poly, fine_nodes[row]))
    return p


# ---------------------------------------------------------------------------
# grid and heat operator  (heat.py:16-158)


@dataclass(frozen=True)
class Op:
    """nu * discrete Laplacian on an interior-only Dirichlet grid."""
    dim: int
    n: int
    nu: float = 1.0
    order: int = 2
    length: float = 1.0

    @property
    def shape(self):
        return (self.n - 1,) * self.dim

    @property
    def dx2(self):
        return (self.length / self.n) ** 2          # heat.py:31-32, 114

    def coarse(self):
        return Op(self.dim, self.n // 2, self.nu, self.order, self.length)


def _shift_axis(u, axis, k, width):
    """u padded with ``width`` zeros on both ends of ``axis``, then sliced so
    that element i holds u[i + k] (zero outside)."""
    pad = [(0, 0)] * u.ndim
    pad[axis] = (width, width)
    up = np.pad(u, pad)
    sl = [slice(None)] * u.ndim
    n = u.shape[axis]
    sl[axis] = slice(width + k, width + k + n)
    return up[tuple(sl)]


def heat_apply(op, u):
    """heat.py:111-142.  Per axis (slowest first) the order-2 term is
    ((u[i-1] - 2u[i]) + u[i+1]) / dx2; the order-4 term is
    ((((-u[i-2] + 16u[i-1]) - 30u[i]) + 16u[i+1]) - u[i+2]) / (12 dx2) with
    the order-2 term at the first/last interior point.  Terms accumulate
    into zeros in axis order; the sum is scaled by nu last."""
    if u.shape != op.shape:
        raise ValueError(f"expected shape {op.shape}, got {u.shape}")
    dx2 = op.dx2
    acc = np.zeros_like(u)
    for ax in range(op.dim):
        w = 1 if op.order == 2 else 2
        m1 = _shift_axis(u, ax, -1, w)
        p1 = _shift_axis(u, ax, 1, w)
        two = (m1 - 2.0 * u + p1) / dx2
        if op.order == 2:
            acc += two
            continue
        m2 = _shift_axis(u, ax, -2, w)
        p2 = _shift_axis(u, ax, 2, w)
        four = (-m2 + 16.0 * m1 - 30.0 * u + 16.0 * p1 - p2) / (12.0 * dx2)
        ends = [slice(None)] * op.dim
        for edge in (slice(0, 1), slice(-1, None)):
            ends[ax] = edge
            four[tuple(ends)] = two[tuple(ends)]
        acc += four
    return op.nu * acc


def heat_diagonal(op):
    """heat.py:144-158."""
    dx2, npts = op.dx2, op.n - 1
    if op.order == 2:
        d1 = np.full(npts, -2.0 / dx2)
    else:
        d1 = np.full(npts, -30.0 / (12.0 * dx2))
        d1[0] = d1[-1] = -2.0 / dx2
    total = np.zeros(op.shape)
    for ax in range(op.dim):
        shp = [1] * op.dim
        shp[ax] = npts
        total = total + d1.reshape(shp)
    return op.nu * total


def shifted_apply(op, sigma, u):
    """multigrid.py:192-193: (I - sigma A) u."""
    return u - sigma * heat_apply(op, u)


@lru_cache(maxsize=None)
def shifted_diag(op, sigma):
    """multigrid.py:186 (computed once per ShiftedOperator in the reference;
    cached here per (operator, sigma) -- same values)."""
    return 1.0 - sigma * heat_diagonal(op)


def operator_matrix(op):
    """Sparse nu*Lap in C order (multigrid.py:86-129)."""
    dx2, npts = op.dx2, op.n - 1
    if op.order == 2:
        d1 = (scipy.sparse.diags([1.0, -2.0, 1.0], [-1, 0, 1],
                                 shape=(npts, npts)) / dx2).tocsr()
    else:
        d1 = scipy.sparse.lil_matrix((npts, npts))
        for i in range(npts):
            if i in (0, npts - 1):
                d1[i, i] = -2.0 / dx2
                for j in (i - 1, i + 1):
                    if 0 <= j < npts:
                        d1[i, j] = 1.0 / dx2
            else:
                for off, w in ((-2, -1.0), (-1, 16.0), (0, -30.0),
                               (1, 16.0), (2, -1.0)):
                    if 0 <= i + off < npts:
                        d1[i, i + off] = w / (12.0 * dx2)
        d1 = d1.tocsr()
    eye = scipy.sparse.identity(npts, format="csr")
    total = None
    for ax in range(op.dim):
        term = None
        for k in range(op.dim):
            f = d1 if k == ax else eye
            term = f if term is None else scipy.sparse.kron(term, f, format="csr")
        total = term if total is None else total + term
    return (op.nu * total).tocsr()


def shifted_matrix(op, sigma):
    """multigrid.py:132-135."""
    a = operator_matrix(op)
    return (scipy.sparse.identity(a.shape[0], format="csr") - sigma * a).tocsr()


def gs_lower_solve_gbtrs(op, sigma, r):
    """(D + L) y = r in the operation order of the reference's
    scipy.linalg.solve_banded (multigrid.py:144-158, 219-224 -> LAPACK
    dgbtrf/dgbtrs, no pivoting since the diagonal dominates each column):
    l_ij = A_ij * RN(1/D_j) (dgbtrf DSCAL), y_i = fma(-y_j, l_ij, y_i) over the
    lower neighbours j in increasing linear index (dgbtrs DGER), du = y / D
    (DTBSV).  Pure-Python loops: the statement the CUDA wavefront
    (csrc/gs.cuh) restates, checked bit for bit against solve_banded in
    tests/test_oracle_golden.py; small grids only."""
    a = shifted_matrix(op, sigma).tocsr()
    d = a.diagonal()
    y = r.ravel().astype(np.float64).copy()
    for i in range(y.size):
        row = a.getrow(i)
        for j, aij in sorted(zip(row.indices, row.data)):
            if j >= i:
                break
            l = aij * (1.0 / d[j])
            y[i] = float(Fraction(-y[j]) * Fraction(l) + Fraction(y[i]))   # exact fma
    return (y / d).reshape(r.shape)


def direct_fast_diag(op, sigma, b):
    """The GPU Direct algorithm (csrc/direct.cu) restated in numpy: T = V
    diag(lam) V^-1 of the 1-D stencil matrix (eigh for order 2, eig + inv for
    order 4), u = (V x..x V) diag(1/(1 - sigma nu sum lam)) (W x..x W) b.
    Equal to the reference's SuperLU solve (multigrid.py:203-208) to
    rounding, not bitwise."""
    npts = op.n - 1
    t = operator_matrix(Op(1, op.n, 1.0, op.order, op.length)).toarray()
    if op.order == 2:
        lam, v = np.linalg.eigh(t)
        w = v.T
    else:
        lam, v = np.linalg.eig(t)
        lam, v = lam.real, v.real
        w = np.linalg.inv(v)
    x = b.copy()
    for ax in range(op.dim):
        x = np.moveaxis(np.tensordot(w, np.moveaxis(x, ax, 0), axes=1), 0, ax)
    s = np.zeros(op.shape)
    for ax in range(op.dim):
        shp = [1] * op.dim
        shp[ax] = npts
        s = s + lam.reshape(shp)
    x = x / (1.0 - sigma * (op.nu * s))
    for ax in range(op.dim):
        x = np.moveaxis(np.tensordot(v, np.moveaxis(x, ax, 0), axes=1), 0, ax)
    return x


# ---------------------------------------------------------------------------
# grid transfers  (transfers.py:19-97)


def _per_axis(u, fn):
    out = u
    for ax in range(u.ndim):
        out = np.moveaxis(fn(np.moveaxis(out, ax, 0)), 0, ax)
    return out


def inject(u):
    """transfers.py:19-24."""
    return _per_axis(u, lambda v: v[1::2])


def full_weighting(u):
    """transfers.py:27-34: 0.25 * ((v[2j-2] + 2 v[2j-1]) + v[2j]) per axis."""
    return _per_axis(u, lambda v: 0.25 * (v[0:-2:2] + 2.0 * v[1:-1:2] + v[2::2]))


def interp_linear(u):
    """transfers.py:37-50."""
    def lin(v):
        out = np.zeros((2 * v.shape[0] + 1,) + v.shape[1:])
        out[1::2] = v
        out[2:-1:2] = 0.5 * (v[:-1] + v[1:])
        out[0] = 0.5 * v[0]
        out[-1] = 0.5 * v[-1]
        return out
    return _per_axis(u, lin)


def cubic_matrix(nf):
    """transfers.py:53-79: 4-tap Lagrange weights through coarse samples,
    boundary samples (index 0 and nc) being zero."""
    nc = nf // 2
    mat = np.zeros((nf - 1, nc - 1))
    for i in range(1, nf):
        if i % 2 == 0:
            mat[i - 1, i // 2 - 1] = 1.0
            continue
        s = i / 2.0
        if nc < 3:
            pts = list(range(0, nc + 1))
        else:
            j0 = min(max(int(np.floor(s)) - 1, 0), nc - 3)
            pts = list(range(j0, j0 + 4))
        for a, ja in enumerate(pts):
            w = 1.0
            for b, jb in enumerate(pts):
                if b != a:
                    w *= (s - jb) / (ja - jb)
            if 1 <= ja <= nc - 1:
                mat[i - 1, ja - 1] += w
    return mat


def interp_cubic(u):
    """transfers.py:82-89 (dense tensordot per axis, as the reference)."""
    out = u
    for ax in range(u.ndim):
        mat = cubic_matrix(2 * (out.shape[ax] + 1))
        out = np.moveaxis(np.tensordot(mat, np.moveaxis(out, ax, 0),
                                       axes=(1, 0)), 0, ax)
    return out


def interp_space(u, order):
    """transfers.py:92-97."""
    if order == 2:
        return interp_linear(u)
    if order == 4:
        return interp_cubic(u)
    raise ValueError("spatial interpolation order must be 2 or 4")


# ---------------------------------------------------------------------------
# multigrid  (multigrid.py:24-288)


@dataclass(frozen=True)
class Mg:
    """multigrid.py:24-38."""
    smoother: str = "jacobi"
    omega: float = 2.0 / 3.0
    pre_sweeps: int = 2
    post_sweeps: int = 2
    coarsest_n: int = 4


@dataclass(frozen=True)
class Fixed:
    """multigrid.py:41-47."""
    cycles: int


@dataclass(frozen=True)
class ToTol:
    """multigrid.py:50-60."""
    tol: float = 1e-12
    stall: float = 0.75
    max_cycles: int = 100


@dataclass(frozen=True)
class DirectSolve:
    """multigrid.py:63-65."""


class MgCapError(RuntimeError):
    """multigrid.py:77-83."""

    def __init__(self, msg, residual, cycles):
        super().__init__(msg)
        self.residual = residual
        self.cycles = cycles


class SubStepFailure(RuntimeError):
    """sdc.py:75-81."""

    def __init__(self, substep, cause):
        super().__init__(f"sub-step {substep}: {cause}")
        self.substep = substep
        self.cause = cause


def red_mask(shape):
    """multigrid.py:167-175: 1-based coordinate sum even."""
    total = np.zeros(shape, dtype=int)
    for ax, npts in enumerate(shape):
        s = [1] * len(shape)
        s[ax] = npts
        total = total + np.arange(1, npts + 1).reshape(s)
    return total % 2 == 0


def smooth(op, sigma, u, b, cfg, count):
    """multigrid.py:211-234."""
    if u.shape != b.shape:
        raise ValueError("shape mismatch between iterate and right-hand side")
    diag = shifted_diag(op, sigma)
    if cfg.smoother == "jacobi":
        for _ in range(count):
            u = u + cfg.omega * (b - shifted_apply(op, sigma, u)) / diag
    elif cfg.smoother == "gauss-seidel":
        lower = scipy.sparse.tril(shifted_matrix(op, sigma), format="coo")
        nb = int(np.max(lower.row - lower.col)) + 1
        ab = np.zeros((nb, lower.shape[0]))
        for k in range(nb):
            d = lower.diagonal(-k)
            ab[k, :d.size] = d
        for _ in range(count):
            r = b - shifted_apply(op, sigma, u)
            du = scipy.linalg.solve_banded((nb - 1, 0), ab, r.ravel())
            u = u + du.reshape(u.shape)
    else:
        red = red_mask(u.shape)
        black = ~red
        u = u.copy()
        for _ in range(count):
            r = b - shifted_apply(op, sigma, u)
            u[red] += cfg.omega * r[red] / diag[red]
            r = b - shifted_apply(op, sigma, u)
            u[black] += cfg.omega * r[black] / diag[black]
    return u


@lru_cache(maxsize=None)
def _coarsest_lu(op, sigma):
    return scipy.linalg.lu_factor(shifted_matrix(op, sigma).toarray())


def coarsest_solve(op, sigma, b):
    """multigrid.py:161-164, 240-243: dense LAPACK LU of I - sigma A
    (factor cached per (operator, sigma) as the reference's lru_cache)."""
    lu = _coarsest_lu(op, sigma)
    return scipy.linalg.lu_solve(lu, b.ravel()).reshape(b.shape)


def v_cycle(op, sigma, u, b, cfg):
    """multigrid.py:237-251."""
    if op.n <= cfg.coarsest_n:
        return coarsest_solve(op, sigma, b)
    u = smooth(op, sigma, u, b, cfg, cfg.pre_sweeps)
    r = b - shifted_apply(op, sigma, u)
    cop = op.coarse()
    ec = v_cycle(cop, sigma, np.zeros(cop.shape), full_weighting(r), cfg)
    u = u + interp_linear(ec)
    return smooth(op, sigma, u, b, cfg, cfg.post_sweeps)


def mg_solve(op, sigma, u0, b, cfg, policy):
    """multigrid.py:261-288 -> (u, cycles, status)."""
    if isinstance(policy, DirectSolve):
        lu = scipy.sparse.linalg.splu(shifted_matrix(op, sigma).tocsc())
        return lu.solve(b.ravel()).reshape(b.shape), 0, "direct"
    if isinstance(policy, Fixed):
        u = u0
        for _ in range(policy.cycles):
            u = v_cycle(op, sigma, u, b, cfg)
        return u, policy.cycles, "fixed"
    bnorm = np.linalg.norm(b.ravel())
    if bnorm == 0.0:
        return np.zeros_like(b), 0, "converged"
    u = u0
    res = np.linalg.norm((b - shifted_apply(op, sigma, u)).ravel())
    cycles = 0
    while res > policy.tol * bnorm:
        if cycles >= policy.max_cycles:
            raise MgCapError(f"no convergence after {cycles} V-cycles "
                             f"(relative residual {res / bnorm:.3e})",
                             res, cycles)
        u = v_cycle(op, sigma, u, b, cfg)
        cycles += 1
        new = np.linalg.norm((b - shifted_apply(op, sigma, u)).ravel())
        if new > policy.tol * bnorm and new >= policy.stall * res:
            return u, cycles, "stalled"
        res = new
    return u, cycles, "converged"


# ---------------------------------------------------------------------------
# SDC  (sdc.py:24-166)


class States:
    """sdc.py:24-47: y, f of shape (M+1, *grid)."""

    def __init__(self, table, y, f):
        self.table, self.y, self.f = table, y, f

    @classmethod
    def spread(cls, op, table, y0):
        f0 = heat_apply(op, y0)
        return cls(table, np.repeat(y0[None], table.m + 1, axis=0),
                   np.repeat(f0[None], table.m + 1, axis=0))

    def copy(self):
        return States(self.table, self.y.copy(), self.f.copy())

    def refresh(self, op):
        for m in range(self.table.m + 1):
            self.f[m] = heat_apply(op, self.y[m])


def sdc_sweep(st, y0, dt, op, cfg, policy, tau=None, solve_log=None):
    """sdc.py:84-114.  ``solve_log`` (oracle-only) collects
    (sigma, cycles, status) per sub-step solve for parity tests."""
    q = st.table.q
    s = dt * np.tensordot(q[1:] - q[:-1], st.f, axes=(1, 0))
    st.y[0] = y0
    st.f[0] = heat_apply(op, y0)
    cycles = 0
    for m in range(st.table.m):
        dtm = float(st.table.gammas[m]) * dt
        rhs = st.y[m] - dtm * st.f[m + 1] + s[m]
        if tau is not None:
            rhs = rhs + (tau[m + 1] - tau[m])
        try:
            u, c, status = mg_solve(op, dtm, st.y[m + 1].copy(), rhs, cfg, policy)
        except MgCapError as exc:
            raise SubStepFailure(m + 1, exc) from exc
        if solve_log is not None:
            solve_log.append((op.n, dtm, c, status))
        st.y[m + 1] = u
        st.f[m + 1] = heat_apply(op, u)
        cycles += c
    return cycles


def residual(st, y0, dt, tau=None):
    """sdc.py:117-124."""
    r = y0[None] + dt * np.tensordot(st.table.q, st.f, axes=(1, 0)) - st.y
    if tau is not None:
        r = r + tau
    return float(np.max(np.abs(r)))


def run_sdc(op, table, u0, t_end, n_steps, tol, max_iter, cfg, policy, solve_log=None):
    """sdc.py:136-166 -> dict(u, iterations, residuals, vcycles, exhausted)."""
    dt = t_end / n_steps
    u = u0
    out = dict(iterations=[], residuals=[], vcycles=0, exhausted=[])
    for step in range(n_steps):
        st = States.spread(op, table, u)
        hist = []
        for _ in range(max_iter):
            out["vcycles"] += sdc_sweep(st, u, dt, op, cfg, policy, solve_log=solve_log)
            hist.append(residual(st, u, dt))
            if hist[-1] <= tol:
                break
        else:
            out["exhausted"].append(step)
        out["iterations"].append(len(hist))
        out["residuals"].append(hist)
        u = st.y[-1].copy()
    out["u"] = u
    return out


# ---------------------------------------------------------------------------
# MLSDC / FAS  (hierarchy.py:27-287)


@dataclass(frozen=True)
class Lvl:
    """hierarchy.py:27-45."""
    op: Op
    table: Table
    cfg: Mg
    policy: object
    interp_order: int = 2
    restrict: str = "full-weighting"


def _restrict(u, fine, coarse):
    """hierarchy.py:66-71."""
    if coarse.op.n == fine.op.n:
        return u.copy()
    if fine.restrict == "inject":
        return inject(u)
    return full_weighting(u)


def _interp(u, fine, coarse):
    """hierarchy.py:74-77."""
    if coarse.op.n == fine.op.n:
        return u
    return interp_space(u, fine.interp_order)


def restrict_state(st, fine, coarse):
    """hierarchy.py:85-93."""
    idx = time_indices(fine.table.nodes, coarse.table.nodes)
    y = np.stack([_restrict(st.y[i], fine, coarse) for i in idx])
    out = States(coarse.table, y, np.empty_like(y))
    out.refresh(coarse.op)
    return out


def compute_fas(fst, cst, fine, coarse, dt, fine_tau=None):
    """hierarchy.py:96-109."""
    fint = dt * np.tensordot(fine.table.q, fst.f, axes=(1, 0))
    if fine_tau is not None:
        fint = fint + fine_tau
    idx = time_indices(fine.table.nodes, coarse.table.nodes)
    rint = np.stack([_restrict(fint[i], fine, coarse) for i in idx])
    return rint - dt * np.tensordot(coarse.table.q, cst.f, axes=(1, 0))


def coarse_correction(fst, old, new, fine, coarse):
    """hierarchy.py:112-122."""
    delta = new.y - old.y
    pt = correction_interp(coarse.table.nodes, fine.table.nodes)
    dtm = np.tensordot(pt, delta, axes=(1, 0))
    for m in range(fine.table.m + 1):
        fst.y[m] = fst.y[m] + _interp(dtm[m], fine, coarse)
    fst.refresh(fine.op)


class Step:
    """hierarchy.py:125-153 (TimeStep)."""

    def __init__(self, levels, states, y0):
        self.levels, self.states, self.y0 = levels, states, y0
        self.tau = [None] * len(levels)

    @classmethod
    def spread(cls, levels, u0):
        states, y0s, u, prev = [], [], u0, None
        for lv in levels:
            if prev is not None:
                u = _restrict(u, prev, lv)
            states.append(States.spread(lv.op, lv.table, u))
            y0s.append(u.copy())
            prev = lv
        return cls(levels, states, y0s)


def _sweep_level(ts, l, dt, log):
    lv = ts.levels[l]
    return sdc_sweep(ts.states[l], ts.y0[l], dt, lv.op, lv.cfg, lv.policy,
                     tau=ts.tau[l], solve_log=log)


def mlsdc_iteration(ts, dt, pre_coarse=None, post_sweep=None, log=None):
    """hierarchy.py:166-203 with the Hooks (hierarchy.py:156-163) as two
    optional callables."""
    L = len(ts.levels)
    if L == 1:
        c = _sweep_level(ts, 0, dt, log)
        if post_sweep:
            post_sweep(0, ts)
        return c
    old = [None] * L
    for l in range(L - 1):
        r = restrict_state(ts.states[l], ts.levels[l], ts.levels[l + 1])
        ts.tau[l + 1] = compute_fas(ts.states[l], r, ts.levels[l],
                                    ts.levels[l + 1], dt, fine_tau=ts.tau[l])
        old[l + 1] = r.copy()
        ts.states[l + 1] = r
        ts.y0[l + 1] = r.y[0].copy()
    if pre_coarse:
        pre_coarse(ts)
    c = _sweep_level(ts, L - 1, dt, log)
    if post_sweep:
        post_sweep(L - 1, ts)
    for l in range(L - 2, -1, -1):
        coarse_correction(ts.states[l], old[l + 1], ts.states[l + 1],
                          ts.levels[l], ts.levels[l + 1])
        ts.y0[l] = ts.states[l].y[0].copy()
        c += _sweep_level(ts, l, dt, log)
        if post_sweep:
            post_sweep(l, ts)
    return c


def burn_in(ts, dt, n, log=None):
    """hierarchy.py:206-219 (no hooks)."""
    return sum(_sweep_level(ts, len(ts.levels) - 1, dt, log) for _ in range(n))


def interpolate_up(ts, spread_copies, exact_y0=None):
    """hierarchy.py:222-238."""
    for l in range(len(ts.levels) - 2, -1, -1):
        coarse_correction(ts.states[l], spread_copies[l + 1], ts.states[l + 1],
                          ts.levels[l], ts.levels[l + 1])
        ts.y0[l] = ts.states[l].y[0].copy()
    if exact_y0 is not None:
        ts.y0[0] = exact_y0.copy()
        ts.states[0].y[0] = exact_y0
        ts.states[0].f[0] = heat_apply(ts.levels[0].op, exact_y0)


def run_mlsdc(levels, u0, t_end, n_steps, tol, max_iter):
    """hierarchy.py:241-287."""
    dt = t_end / n_steps
    u = u0
    out = dict(iterations=[], residuals=[], vcycles=0, exhausted=[])
    for step in range(n_steps):
        ts = Step.spread(levels, u)
        if len(levels) > 1:
            copies = [s.copy() for s in ts.states]
            out["vcycles"] += burn_in(ts, dt, 1)
            interpolate_up(ts, copies, exact_y0=u)
        hist = []
        for _ in range(max_iter):
            out["vcycles"] += mlsdc_iteration(ts, dt)
            hist.append(residual(ts.states[0], ts.y0[0], dt))
            if hist[-1] <= tol:
                break
        else:
            out["exhausted"].append(step)
        out["iterations"].append(len(hist))
        out["residuals"].append(hist)
        u = ts.states[0].y[-1].copy()
    out["u"] = u
    return out


# ---------------------------------------------------------------------------
# PFASST, serial (normative) schedule  (pfasst.py:121-287)


@dataclass
class PfasstOut:
    u: np.ndarray
    rank_iterations: list = field(default_factory=list)
    rank_vcycles: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    trace: list = field(default_factory=list)      # (block, rank, it, level, res, cyc)
    final_values: list = field(default_factory=list)
    solve_log: list = field(default_factory=list)  # oracle-only parity aid


def pfasst_run(levels, u0, t_end, p, blocks=1, tol=1e-9, max_iter=20,
               record_final_values=False, log_solves=False):
    """pfasst.py:256-287 with _run_block_serial (pfasst.py:213-228)."""
    if p < 1 or blocks < 1:
        raise ValueError("need at least one rank and one block")
    dt = t_end / (p * blocks)
    L = len(levels)
    c = L - 1
    out = PfasstOut(u=u0)
    u = u0
    for block in range(blocks):
        log = [] if log_solves else None
        board = {}
        steps = [Step.spread(levels, u) for _ in range(p)]
        copies = [[s.copy() for s in ts.states] for ts in steps]
        vcyc, iters, conv = [0] * p, [0] * p, [False] * p
        frozen_payload = [dict() for _ in range(p)]
        trace, finals = [], []

        def send(rank, level, tag, payload):          # pfasst.py:144-148
            snap = payload.copy()
            frozen_payload[rank][level] = snap
            if rank + 1 < p:
                board[(rank, level, tag)] = snap

        # predictor (pfasst.py:166-176, 215-217)
        for ph in range(p):
            for n in range(ph, p):
                ts = steps[n]
                if n > 0:
                    ts.y0[c] = board[(n - 1, c, ("pred", min(ph, n - 1)))]
                vcyc[n] += burn_in(ts, dt, 1, log)
                if n + 1 < p:
                    board[(n, c, ("pred", ph))] = ts.states[c].y[-1].copy()
        for n in range(p):                            # pfasst.py:178-181
            interpolate_up(steps[n], copies[n],
                           exact_y0=steps[n].y0[0] if n == 0 else None)
        frozen = [False] * p
        for k in range(1, max_iter + 1):
            for n in range(p):
                if frozen[n]:                         # pfasst.py:156-162
                    if n + 1 < p:
                        for lvl, pay in frozen_payload[n].items():
                            board[(n, lvl, ("it", k))] = \
                                (pay, True) if lvl == 0 else pay
                    continue
                ts = steps[n]
                pred_ok = n == 0
                if n > 0:                             # pfasst.py:189-198
                    for lvl in range(L - 1):
                        msg = board[(n - 1, lvl, ("it", k))]
                        if lvl == 0:
                            pay, pred_ok = msg
                        else:
                            pay = msg
                        ts.y0[lvl] = pay
                        ts.states[lvl].y[0] = pay
                        ts.states[lvl].f[0] = heat_apply(levels[lvl].op, pay)

                def pre(ts_, n=n, k=k):               # pfasst.py:107-112
                    if n > 0:
                        ts_.y0[c] = board[(n - 1, c, ("it", k))]

                def post(l, ts_, n=n, k=k):           # pfasst.py:114-118
                    if l != 0:
                        send(n, l, ("it", k), ts_.states[l].y[-1])

                cyc = mlsdc_iteration(ts, dt, pre, post, log)
                res = residual(ts.states[0], ts.y0[0], dt)
                ok = res <= tol and pred_ok
                snap = ts.states[0].y[-1].copy()      # pfasst.py:150-154
                frozen_payload[n][0] = snap
                if n + 1 < p:
                    board[(n, 0, ("it", k))] = (snap, ok)
                vcyc[n] += cyc
                iters[n] = k
                conv[n] = ok
                trace.append((block, n, k, 0, res, cyc))
                if record_final_values and n == p - 1:
                    finals.append(ts.states[0].y[-1].copy())
                frozen[n] = ok
            if frozen[-1]:
                break
        u = steps[-1].states[0].y[-1].copy()
        out.rank_iterations.append(list(iters))
        out.rank_vcycles.append(list(vcyc))
        out.converged.append(list(conv))
        out.trace.extend(sorted(trace, key=lambda r: (r[2], r[1], r[3])))
        out.final_values.append(finals)
        if log is not None:
            out.solve_log.append(log)
    out.u = u
    return out


# ---------------------------------------------------------------------------
# synthetic inputs


def sine_mode(dim, n, k, length=1.0):
    """heat.py:55-62: product of sin(k pi x / L) at interior points."""
    x = (length / n) * np.arange(1, n)
    axis = np.sin(k * np.pi * x / length)
    u = axis
    for _ in range(dim - 1):
        u = np.multiply.outer(u, axis)
    return u


def seeded_field(dim, n, seed=1407, modes=16, kmax=32, amp=1e-2, length=1.0):
    """sin-product base mode plus ``modes`` seeded Fourier modes (SURVEY.md
    8(d)): for each mode j in order, k_j = rng.integers(1, kmax+1, size=dim)
    then a_j = rng.uniform(0, amp); axis 0 uses k_j[0].  Each axis factor is
    sampled like heat.py:55-62 (sin(k pi x / L), x = dx * (1..n-1))."""
    rng = np.random.default_rng(seed)
    x = (length / n) * np.arange(1, n)
    u = sine_mode(dim, n, 1, length)
    for _ in range(modes):
        k = rng.integers(1, kmax + 1, size=dim)
        a = rng.uniform(0, amp)
        term = np.sin(int(k[0]) * np.pi * x / length)
        for d in range(1, dim):
            term = np.multiply.outer(term, np.sin(int(k[d]) * np.pi * x / length))
        u = u + a * term
    return u
