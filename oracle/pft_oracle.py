"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference hot path.

A CPU oracle for the parity tests, written from the reference's algorithm
(/root/reference/proj/core/src, cited per function as file:line). It follows
the reference's stage order; numpy supplies the GEMMs (Eigen in the reference)
and the FFTs (FFTW in the reference). Pinned against the golden fixtures in
tests/golden (produced by the reference itself, oracle/_ref) and against
oracle/_ref directly where that is built (tests/test_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module. The product (libpftg + paper_2408_03532_b200) never does.
"""
from __future__ import annotations

import dataclasses
from pathlib import Path

import numpy as np

KPI = 3.14159265358979323846  # pft.cpp:17


# ---------------------------------------------------------------- scope table
@dataclasses.dataclass
class Record:
    eps: float
    r: int
    xi: float
    achieved_error: float
    coeff: np.ndarray  # complex128, length r


def load_scope_table(path) -> list[Record]:
    """ScopeTable::load (minimax.cpp:495-522): 'pft-scope-table v1' records."""
    lines = Path(path).read_text().splitlines()
    if not lines or lines[0] != "pft-scope-table v1":
        raise RuntimeError(f"ScopeTable: bad header in {path}")
    recs = []
    for ln in lines[1:]:
        if not ln or ln.startswith("#"):
            continue
        tok = ln.split()
        if tok[0] != "record":
            raise RuntimeError("ScopeTable: malformed record line")
        eps, r, xi, ach = float(tok[1]), int(tok[2]), float(tok[3]), float(tok[4])
        vals = np.array([float(v) for v in tok[5:5 + 2 * r]])
        recs.append(Record(eps, r, xi, ach, vals[0::2] + 1j * vals[1::2]))
    return recs


def find_record(table, eps, r):
    """ScopeTable::find (minimax.cpp:435-439): relative eps match 1e-9."""
    for rec in table:
        if rec.r == r and abs(rec.eps - eps) <= 1e-9 * eps:
            return rec
    return None


def min_degree(table, eps, target):
    """ScopeTable::min_degree (minimax.cpp:455-468)."""
    max_r = max(rec.r for rec in table)
    best = 0.0
    for r in range(1, max_r + 1):
        rec = find_record(table, eps, r)
        if rec is None:
            continue
        best = max(best, rec.xi)
        if rec.xi >= target:
            return r
    raise ValueError(f"min_degree: target scope {target} infeasible for eps {eps} "
                     f"(best achievable {best})")


# ---------------------------------------------------------------- plans
@dataclasses.dataclass
class Axis:
    n: int
    p: int
    q: int
    mt: int
    r: int
    eps: float
    B: np.ndarray  # q x r
    W: np.ndarray  # (2mt+1) x r


def plan_1d(n, mt, p, eps, table) -> Axis:
    """pft_plan_1d (pft.cpp:33-76): B[l,j] = w_j x_l^j, W[i,j] = e^{-i pi t/p} (t/p)^j."""
    if p < 2 or p > n or n % p:
        raise ValueError("pft_plan_1d: p must divide n, 2 <= p <= n")
    q = n // p
    if q < 2:
        raise ValueError("pft_plan_1d: need q = n/p >= 2")
    if mt < 1 or 2 * mt > n:
        raise ValueError("pft_plan_1d: need 1 <= mt and 2*mt <= n")
    r = min_degree(table, eps, mt / p)
    w = find_record(table, eps, r).coeff
    B = np.empty((q, r), np.complex128)
    for l in range(q):
        x = 1.0 - 2.0 * l / q
        xpow = 1.0
        for j in range(r):  # repeated multiplication, as the reference
            B[l, j] = w[j] * xpow
            xpow *= x
    W = np.empty((2 * mt + 1, r), np.complex128)
    for i in range(2 * mt + 1):
        base = (i - mt) / p
        tw = complex(np.cos(-KPI * base), np.sin(-KPI * base))
        bpow = 1.0
        for j in range(r):
            W[i, j] = tw * bpow
            bpow *= base
    return Axis(n, p, q, mt, r, eps, B, W)


def pft_apply_1d(a: Axis, z, dtype=np.complex128):
    """pft_apply_1d (pft.cpp:78-101): C = reshape(z, p x q) B, column FFTs over
    k (FFTW_FORWARD), out[i] = sum_j C[(i - mt) mod p, j] W[i, j], i in [0, 2mt]."""
    ct = _ctype(dtype)
    z = np.asarray(z).astype(ct).reshape(a.p, a.q)
    Cm = z @ a.B.astype(ct)
    Cm = np.fft.fft(Cm, axis=0).astype(ct)
    u = (np.arange(2 * a.mt + 1) - a.mt) % a.p
    return np.sum(Cm[u, :] * a.W.astype(ct), axis=1)


@dataclasses.dataclass
class Plan2D:
    a1: Axis
    a2: Axis


def plan_2d(n1, n2, mt1, mt2, p1, p2, eps, table) -> Plan2D:
    """pft_plan_2d (pft.cpp:103-112)."""
    return Plan2D(plan_1d(n1, mt1, p1, eps, table), plan_1d(n2, mt2, p2, eps, table))


def _u(M, mt, p):
    """u = (a - mt) mod p, non-negative (pft.cpp:25-29)."""
    return (np.arange(M) - mt) % p


def _ctype(dtype):
    """oracle<double> (complex128, the default) or oracle<float> (complex64):
    every stage below runs in that precision -- tables rounded once, products and
    sums (einsum), the slice DFT (numpy.fft keeps complex64) -- so the float
    variant measures the deviation an exact-order single-precision evaluation of
    the reference's algorithm has from the double one (the complex64 parity floor,
    SURVEY §8(c) C5)."""
    ct = np.dtype(dtype)
    if ct not in (np.complex64, np.complex128):
        raise TypeError("oracle dtype must be complex64 or complex128")
    return ct


def pft_apply_2d(plan: Plan2D, z, dtype=np.complex128):
    """pft_apply_2d (pft.cpp:119-172), same four stages in the same order."""
    a1, a2 = plan.a1, plan.a2
    ct = _ctype(dtype)
    z = np.asarray(z).astype(ct)
    if z.shape != (a1.n, a2.n):
        raise ValueError("pft_apply_2d: z shape must match the plan")
    B1, B2 = a1.B.astype(ct), a2.B.astype(ct)
    W1, W2 = a1.W[: 2 * a1.mt].astype(ct), a2.W[: 2 * a2.mt].astype(ct)
    Z = z.reshape(a1.p, a1.q, a2.n)
    # stage A (133-136): T[k1] = B1^T Z_blk
    T = np.einsum("lj,kln->kjn", B1, Z)
    # stage B (137-144): C[k1,k2,j1,j2] = sum_l2 T[k1,j1,k2*q2+l2] B2[l2,j2]
    C = np.einsum("kjpl,lm->kpjm", T.reshape(a1.p, a1.r, a2.p, a2.q), B2)
    # stage C (147): unnormalized 2-D DFT over (k1, k2)
    Ch = np.fft.fft2(C, axes=(0, 1))
    # stage D (149-170): out[a,b] = sum_j1 W1[a,j1] sum_j2 Ch[u1,u2,j1,j2] W2[b,j2]
    u1, u2 = _u(2 * a1.mt, a1.mt, a1.p), _u(2 * a2.mt, a2.mt, a2.p)
    S = Ch[u1][:, u2]  # (M1, M2, r1, r2)
    inner = np.einsum("abjm,bm->abj", S, W2)
    return np.einsum("aj,abj->ab", W1, inner)


def pft_adjoint_2d(plan: Plan2D, band, dtype=np.complex128):
    """pft_adjoint_2d (pft.cpp:174-226): D-dagger scatter, backward DFT, B-dagger, A-dagger.
    ``dtype`` as in pft_apply_2d (complex64 = oracle<float>)."""
    a1, a2 = plan.a1, plan.a2
    ct = _ctype(dtype)
    y = np.asarray(band).astype(ct)
    if y.shape != (2 * a1.mt, 2 * a2.mt):
        raise ValueError("pft_adjoint_2d: band shape must match the plan")
    W1c = np.conj(a1.W[: 2 * a1.mt]).astype(ct)
    W2c = np.conj(a2.W[: 2 * a2.mt]).astype(ct)
    u1, u2 = _u(2 * a1.mt, a1.mt, a1.p), _u(2 * a2.mt, a2.mt, a2.p)
    # D-dagger: contribution of band element (a, b) to (u1, u2, j1, j2), in the
    # reference's order c1 = conj(W1[a,j1]) y(a,b), then c1 conj(W2[b,j2]) (184-203)
    c1 = np.einsum("aj,ab->abj", W1c, y)
    contrib = np.einsum("abj,bm->abjm", c1, W2c)
    C = np.zeros((a1.p, a2.p, a1.r, a2.r), ct)
    np.add.at(C, (u1[:, None], u2[None, :]), contrib)  # scatter-accumulate (184-203)
    C = (np.fft.ifft2(C, axes=(0, 1)) * (a1.p * a2.p)).astype(ct)  # unnormalized backward (205)
    M = np.einsum("kpjm,lm->kjpl", C, np.conj(a2.B).astype(ct))  # M = Cslice B2^H (213-220)
    T = M.reshape(a1.p, a1.r, a2.n)
    Z = np.einsum("lj,kjn->kln", np.conj(a1.B).astype(ct), T)  # Zblk = conj(B1) T (221-223)
    return Z.reshape(a1.n, a2.n)


# ---------------------------------------------------------------- transforms
def fast_fft2(z, dtype=np.complex128):
    """fast_fft2 (fft.cpp:175-178): unnormalized forward."""
    return np.fft.fft2(np.asarray(z).astype(_ctype(dtype)))


def fast_ifft2(z, dtype=np.complex128):
    """fast_ifft2 (fft.cpp:180-183): inverse with 1/n."""
    return np.fft.ifft2(np.asarray(z).astype(_ctype(dtype)))


def naive_dft2(z):
    """naive_dft2 (fft.cpp:132-146), exact integer phase reduction; small n only."""
    z = np.asarray(z, np.complex128)
    n1, n2 = z.shape
    k1, k2 = np.arange(n1), np.arange(n2)
    F1 = np.exp(-2j * np.pi * ((np.outer(k1, k1) % n1) / n1))
    F2 = np.exp(-2j * np.pi * ((np.outer(k2, k2) % n2) / n2))
    return F1 @ z @ F2.T


def crop_centered(spectrum, mt1, mt2):
    """crop_centered (fft.cpp:206-232): out(a,b) = s((a-mt1) mod n1, (b-mt2) mod n2)."""
    s = np.asarray(spectrum)
    n1, n2 = s.shape
    if mt1 == 0 or mt2 == 0:
        raise ValueError("crop_centered: mt must be >= 1")
    if 2 * mt1 > n1 or 2 * mt2 > n2:
        raise ValueError("crop_centered: band exceeds spectrum shape")
    return s[np.ix_(_u(2 * mt1, mt1, n1), _u(2 * mt2, mt2, n2))]


def _phase_unit(v):
    """phase_unit (solver.cpp:21-24): v/|v|, 1 where |v| == 0."""
    a = np.abs(v)
    out = np.ones_like(v)
    nz = a > 0
    out[nz] = v[nz] / a[nz]
    return out


def project_modulus(exit_wave, d, dtype=np.complex128):
    """project_modulus (solver.cpp:35-42)."""
    spec = fast_fft2(exit_wave, dtype)
    return fast_ifft2(np.asarray(d).astype(spec.real.dtype) * _phase_unit(spec), dtype)


def band_residual(plan, exit_wave, d_crop, dtype=np.complex128):
    """band_residual (solver.cpp:61-69)."""
    band = pft_apply_2d(plan, exit_wave, dtype)
    return pft_adjoint_2d(plan, band - np.asarray(d_crop).astype(band.real.dtype) * _phase_unit(band),
                          dtype)


def pie_object_update(zj, probe, projected, beta):
    """pie_object_update (solver.cpp:44-50), returns the new patch."""
    return zj - beta * np.conj(probe) * (probe * zj - projected)


def epie_probe_update(probe, zj, projected, gamma, blind=True):
    """epie_probe_update (solver.cpp:52-59), returns the new probe."""
    if not blind:
        raise RuntimeError("epie_probe_update: probe updates need blind mode")
    return probe - gamma * np.conj(zj) * (probe * zj - projected)


def objective_value(frame, probe, offsets, d, dtype=np.complex128):
    """objective_value (solver.cpp:89-102)."""
    wr, wc = probe.shape
    acc = 0.0
    for j, (r0, c0) in enumerate(offsets):
        ex = frame[r0:r0 + wr, c0:c0 + wc] * probe
        acc += float(np.sum(np.abs(ex - project_modulus(ex, d[j], dtype)).astype(np.float64) ** 2))
    return acc / len(offsets)


def evaluate_shard(frame, probe, offsets, d, begin, end):
    """Unnormalized objective numerator over positions [begin, end) (the
    per-rank partial of the sharded evaluator; summed across ranks then / N)."""
    wr, wc = probe.shape
    acc = 0.0
    for j in range(begin, end):
        r0, c0 = offsets[j]
        ex = frame[r0:r0 + wr, c0:c0 + wc] * probe
        acc += float(np.sum(np.abs(ex - project_modulus(ex, d[j])) ** 2))
    return acc


class Mt19937_64:
    """std::mt19937_64 (the C++ standard's parameters; default-seeded like
    ``std::mt19937_64 rng(seed)``), for the shuffled visit order."""

    def __init__(self, seed):
        m = (1 << 64) - 1
        self.mt = [seed & m]
        for i in range(1, 312):
            prev = self.mt[-1]
            self.mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & m)
        self.i = 312

    def __call__(self):
        m = (1 << 64) - 1
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & m


def shuffle_order(order, rng):
    """shuffle_order (solver.cpp:164-169): Fisher-Yates with rng() % i draws."""
    for i in range(len(order), 1, -1):
        j = rng() % i
        order[i - 1], order[j] = order[j], order[i - 1]


def tv_gradient(x):
    """tv_gradient (solver.cpp:71-87): psi'(t) = t / sqrt(t^2 + 1e-12) over the
    4-neighbourhood, one-sided at the edges, accumulated in the reference's order."""
    x = np.asarray(x, np.float64)
    psi = lambda t: t / np.sqrt(t * t + 1e-6 * 1e-6)  # noqa: E731
    g = np.zeros_like(x)
    dv = psi(x[1:, :] - x[:-1, :])  # dv[i] = psi(x[i+1] - x[i])
    dh = psi(x[:, 1:] - x[:, :-1])
    g[:-1, :] -= dv
    g[1:, :] += dv
    g[:, :-1] -= dh
    g[:, 1:] += dh
    return g


def tv_step(frame, lam_mag, lam_phase, step):
    """The per-sweep TV block of hybrid_solve (solver.cpp:264-279): magnitude /
    phase (phase of 0 is 0, field.cpp:74-87), gradient steps, from_polar."""
    mag = np.abs(frame).astype(np.float64)
    ph = np.where(frame == 0, 0.0, np.angle(frame)).astype(np.float64)
    if lam_mag > 0:
        mag = mag - lam_mag * step * tv_gradient(mag)
    if lam_phase > 0:
        ph = ph - lam_phase * step * tv_gradient(ph)
    return (mag * np.cos(ph) + 1j * (mag * np.sin(ph))).astype(frame.dtype)


def hybrid_solve(frame, probe, offsets, d, *, pft_sweeps, fft_sweeps, table=None, beta=1.0,
                 gamma=1.0, beta_pft=1e-3, gamma_pft=1e-3, eps_pft=1e-3, mt=0, p=0, blind=False,
                 shuffled=False, seed=0, dtype=np.complex128, tv_mag=0.0, tv_phase=0.0):
    """hybrid_solve (solver.cpp:173-302), tol = 0; TV (264-279) when tv_mag /
    tv_phase > 0.
    ``dtype=np.complex64`` is oracle<float>: frame, probe, measurements and every
    operator in single precision (the reference of the complex64 ePIE tolerance).

    Returns (frame, probe, objectives)."""
    ct = _ctype(dtype)
    rt = np.float32 if ct == np.complex64 else np.float64
    frame = np.array(frame).astype(ct)
    probe = np.array(probe).astype(ct)
    d = np.asarray(d).astype(rt)
    beta, gamma, beta_pft, gamma_pft = (rt(v) for v in (beta, gamma, beta_pft, gamma_pft))
    wr, wc = probe.shape
    plan = dcrop = None
    if pft_sweeps > 0:
        mt1 = mt or wr // 8
        mt2 = mt or wc // 8
        p1, p2 = (p or mt1), (p or mt2)
        plan = plan_2d(wr, wc, mt1, mt2, p1, p2, eps_pft, table)
        dcrop = [crop_centered(dj, mt1, mt2) for dj in d]
    objs = []
    rng = Mt19937_64(seed)
    order = list(range(len(offsets)))
    for sweep in range(1, pft_sweeps + fft_sweeps + 1):
        band_stage = sweep <= pft_sweeps
        if shuffled:  # solver.cpp:222-236, the order persists across sweeps
            shuffle_order(order, rng)
        for j in order:
            r0, c0 = offsets[j]
            zj = frame[r0:r0 + wr, c0:c0 + wc].copy()
            ex = probe * zj
            if band_stage:
                zj = zj - beta_pft * np.conj(probe) * band_residual(plan, ex, dcrop[j], ct)
                if blind:
                    resid2 = band_residual(plan, probe * zj, dcrop[j], ct)
                    probe = probe - gamma_pft * np.conj(zj) * resid2
            else:
                zj = pie_object_update(zj, probe, project_modulus(ex, d[j], ct), beta)
                if blind:
                    probe = epie_probe_update(probe, zj, project_modulus(probe * zj, d[j], ct), gamma)
            frame[r0:r0 + wr, c0:c0 + wc] = zj
        if tv_mag > 0 or tv_phase > 0:
            frame = tv_step(frame, tv_mag, tv_phase, float(beta_pft if band_stage else beta))
        objs.append(objective_value(frame, probe, offsets, d, ct))
    return frame, probe, np.array(objs)
