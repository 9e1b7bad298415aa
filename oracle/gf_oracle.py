"""CPU ORACLE for the matrix-free contraction engine -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the timed CPU port -- never as the thing measured or shipped.

It restates the reference package ``gatefit`` (arXiv 2506.23775):

* ``gf_oracle.c`` holds the numba cores and per-summand drivers in plain C
  (reference kernels.py:132-458, objective.py:255-482);
* this module restates the host glue: the circuit plan (objective.py:157-199),
  pair CSR (objective.py:209-247), fixed 64-state chunks combined in ascending
  order (objective.py:490-533), logical accumulation (objective.py:645-647,
  circuit.py:161-170), the spinful / spinless Fermi-Hubbard term lists
  (models.py:94-170), the dense target (models.py:258-319) and the Lanczos
  target (models.py:322-384).

Parity: PINNED against fixtures from the unmodified reference
(tests/golden/make_golden.py -> tests/test_oracle.py).  Sector / fold sums have
no reference implementation; they are pinned through the reference drivers run
over the restricted index sets (same fixtures).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "_build", "libgforacle.so")

WIRE_SWAP = np.array([0, 2, 1, 3])
DENSE_SUPPORT = np.arange(16)
PARITY_SUPPORT = np.array([0, 3, 5, 6, 9, 10, 12, 15])
CHUNK_STATES = 64  # reference objective.py:75


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load():
    if not os.path.exists(_SO):
        build()
    return ctypes.CDLL(_SO)


_lib = _load()
_P = ctypes.c_void_p
_I = ctypes.c_int64


class _Plan(ctypes.Structure):
    _fields_ = [("k", _I), ("nslots", _I), ("mats", _P), ("mats_t", _P), ("sparse", _P),
                ("ps", _P), ("qs", _P), ("ns", _P)]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def leg_dims(k, q1, q2):
    return 2**q1, 2 ** (q2 - q1 - 1), 2 ** (k - 1 - q2)


def swap_wires(m):
    return np.ascontiguousarray(m[WIRE_SWAP][:, WIRE_SWAP])


def swapped_support(sup):
    sup = np.asarray(sup)
    return WIRE_SWAP[sup // 4] * 4 + WIRE_SWAP[sup % 4]


def _norm(k, targets):
    t1, t2 = int(targets[0]), int(targets[1])
    if t1 == t2 or not (0 <= t1 < k and 0 <= t2 < k):
        raise ValueError("bad targets")
    return (t1, t2, False) if t1 < t2 else (t2, t1, True)


# ---------------------------------------------------------------- kernels


def apply_gate(psi, g, targets, sparse=False):
    psi = _c(psi)
    k = int(np.log2(psi.size))
    q1, q2, sw = _norm(k, targets)
    g = _c(g)
    if sw:
        g = swap_wires(g)
    p, q, n = leg_dims(k, q1, q2)
    out = np.empty_like(psi)
    _lib.or_apply(_ptr(psi), _ptr(g), _I(p), _I(q), _I(n), ctypes.c_int(int(sparse)), _ptr(out))
    return out


def hole_contract(bra, ket, targets):
    bra, ket = _c(bra), _c(ket)
    k = int(np.log2(bra.size))
    q1, q2, sw = _norm(k, targets)
    p, q, n = leg_dims(k, q1, q2)
    out = np.empty(16, np.complex128)
    _lib.or_hole_contract(_ptr(bra), _ptr(ket), _I(p), _I(q), _I(n), _ptr(out))
    out = out.reshape(4, 4)
    return swap_wires(out) if sw else out


def hole_apply(psi, targets, support=None):
    psi = _c(psi)
    k = int(np.log2(psi.size))
    q1, q2, sw = _norm(k, targets)
    sup = DENSE_SUPPORT if support is None else np.asarray(support)
    eff = swapped_support(sup) if sw else sup
    rows, cols = np.ascontiguousarray(eff // 4, np.int64), np.ascontiguousarray(eff % 4, np.int64)
    p, q, n = leg_dims(k, q1, q2)
    out = np.empty((psi.size, len(sup)), np.complex128)
    _lib.or_hole_apply(_ptr(psi), _I(p), _I(q), _I(n), _ptr(rows), _ptr(cols), _I(len(sup)), _ptr(out))
    return out


def apply_gate_to_array(arr, g, targets, sparse=False):
    arr = _c(arr)
    k = int(np.log2(arr.shape[0]))
    q1, q2, sw = _norm(k, targets)
    g = _c(g)
    if sw:
        g = swap_wires(g)
    p, q, n = leg_dims(k, q1, q2)
    out = np.empty_like(arr)
    _lib.or_array_apply(_ptr(arr), _I(arr.shape[1]), _ptr(g), _I(p), _I(q), _I(n), ctypes.c_int(int(sparse)),
                        _ptr(out))
    return out


def hole_contract_array(bra, arr, targets, support=None):
    bra, arr = _c(bra), _c(arr)
    k = int(np.log2(bra.size))
    q1, q2, sw = _norm(k, targets)
    sup = DENSE_SUPPORT if support is None else np.asarray(support)
    eff = swapped_support(sup) if sw else sup
    rows, cols = np.ascontiguousarray(eff // 4, np.int64), np.ascontiguousarray(eff % 4, np.int64)
    p, q, n = leg_dims(k, q1, q2)
    outT = np.empty((len(sup), arr.shape[1]), np.complex128)
    _lib.or_hole_contract_array(_ptr(bra), _ptr(arr), _I(arr.shape[1]), _I(p), _I(q), _I(n), _ptr(rows),
                                _ptr(cols), _I(len(sup)), _ptr(outT))
    return np.ascontiguousarray(outT.T)


# ---------------------------------------------------------------- plan


class Plan:
    """Restates objective._Plan (reference objective.py:157-199)."""

    def __init__(self, k, targets, logical, gates, parity_mode=False):
        targets = np.asarray(targets, np.int64).reshape(-1, 2)
        self.k = k
        self.n = n = len(targets)
        self.logical = np.asarray(logical, np.int64)
        self.nlog = len(gates)
        self.support = PARITY_SUPPORT if parity_mode else DENSE_SUPPORT
        A = len(self.support)
        self.mats = np.empty((n, 16), np.complex128)
        self.mats_t = np.empty((n, 16), np.complex128)
        self.sparse = np.zeros(n, np.int32)
        self.ps, self.qs, self.ns = (np.empty(n, np.int64) for _ in range(3))
        self.swapped = np.zeros(n, bool)
        self.hole_row = np.empty((n, A), np.int64)
        self.hole_col = np.empty((n, A), np.int64)
        self.targets = targets
        for i, (t1, t2) in enumerate(targets):
            q1, q2, sw = _norm(k, (t1, t2))
            m = _c(gates[self.logical[i]])
            if sw:
                m = swap_wires(m)
            self.mats[i] = m.reshape(16)
            self.mats_t[i] = m.T.reshape(16)
            off = m.reshape(16)[[1, 2, 4, 7, 8, 11, 13, 14]]
            self.sparse[i] = int(parity_mode and np.all(off == 0))
            self.ps[i], self.qs[i], self.ns[i] = leg_dims(k, q1, q2)
            self.swapped[i] = sw
            sup = swapped_support(self.support) if sw else self.support
            self.hole_row[i], self.hole_col[i] = sup // 4, sup % 4
        self._c = _Plan(k, n, _ptr(self.mats), _ptr(self.mats_t), _ptr(self.sparse), _ptr(self.ps), _ptr(self.qs),
                        _ptr(self.ns))

    def unswap(self, d, i):
        return swap_wires(d) if self.swapped[i] else d

    def logical_sum(self, per_slot):
        """Unswap + accumulate onto logical gates (objective.py:645-647)."""
        out = np.zeros((self.nlog, 4, 4), np.complex128)
        for i in range(self.n):
            out[self.logical[i]] += self.unswap(per_slot[i].reshape(4, 4), i)
        return out

    def zmats(self, directions):
        zm = np.empty((self.n, 16), np.complex128)
        zt = np.empty((self.n, 16), np.complex128)
        for i in range(self.n):
            z = _c(directions[self.logical[i]])
            if self.swapped[i]:
                z = swap_wires(z)
            zm[i], zt[i] = z.reshape(16), z.T.reshape(16)
        return zm, zt


def pair_csr(targets, logical, nlog, classes=None):
    """Restates objective._pair_csr (objective.py:209-247); ``classes`` is a
    list of ((a, b), multiplicity) from translation classes, else all pairs."""
    n = len(logical)
    if classes is None:
        classes = [((a, b), 1) for a in range(n) for b in range(a + 1, n)]
    grouped = {}
    for (a, b), m in classes:
        grouped.setdefault(a, []).append((b, m))
    firsts = sorted(grouped)
    starts, sec, mult, route, sym, flip = [0], [], [], [], [], []
    for a in firsts:
        for b, m in sorted(grouped[a]):
            la, lb = int(logical[a]), int(logical[b])
            lo, hi = min(la, lb), max(la, lb)
            sec.append(b)
            mult.append(float(m))
            route.append(lo * nlog - lo * (lo - 1) // 2 + (hi - lo))
            sym.append(la == lb)
            flip.append(la > lb)
        starts.append(len(sec))
    return (np.array(firsts, np.int64), np.array(starts, np.int64), np.array(sec, np.int64),
            np.array(mult, np.float64), np.array(route, np.int64), np.array(sym, np.int32),
            np.array(flip, np.int32))


# ---------------------------------------------------------------- basis sums


def chunk_bounds(total, size=CHUNK_STATES):
    """objective.py:490-510: chunk count = total // 64 (>= 1), near-equal."""
    if total == 0:
        return []
    nch = max(1, min(total // size, total))
    base, extra = divmod(total, nch)
    out, s = [], 0
    for c in range(nch):
        e = s + base + (1 if c < extra else 0)
        out.append((s, e))
        s = e
    return out


def _reduce(js, fn, workers):
    bounds = chunk_bounds(len(js))
    if workers <= 1:
        parts = [fn(js[a:b]) for a, b in bounds]
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(lambda ab: fn(js[ab[0]:ab[1]]), bounds))
    acc = parts[0]
    for p in parts[1:]:
        acc = tuple(x + y for x, y in zip(acc, p))
    return acc


def value_sum(plan, js, phi0_fn, workers=1):
    """Sum over js of phi0(j) . C|j>  (objective.py:291-304)."""
    js = np.asarray(js, np.int64)
    N = 2**plan.k

    def fn(jj):
        phi = _c(phi0_fn(jj))
        a, b = np.empty(N, np.complex128), np.empty(N, np.complex128)
        counts = np.zeros(5, np.int64)
        v = np.zeros(1, np.complex128)
        jj = np.ascontiguousarray(jj)
        _lib.or_value_chunk(ctypes.byref(plan._c), _ptr(jj), _I(len(jj)), _ptr(phi), _ptr(a), _ptr(b),
                            _ptr(counts), _ptr(v))
        return v[0], counts

    return _reduce(js, fn, workers)


def gradient_sum(plan, js, phi0_fn, workers=1):
    """(value, per-slot D [n,16], counts) (objective.py:322-337)."""
    js = np.asarray(js, np.int64)
    N, n = 2**plan.k, plan.n

    def fn(jj):
        phi = _c(phi0_fn(jj))
        psis = np.empty((n + 1, N), np.complex128)
        phis = np.empty((n + 1, N), np.complex128)
        dacc = np.zeros((n, 16), np.complex128)
        counts = np.zeros(5, np.int64)
        v = np.zeros(1, np.complex128)
        jj = np.ascontiguousarray(jj)
        _lib.or_gradient_chunk(ctypes.byref(plan._c), _ptr(jj), _I(len(jj)), _ptr(phi), _ptr(psis), _ptr(phis),
                               _ptr(dacc), _ptr(counts), _ptr(v))
        return v[0], dacc, counts

    return _reduce(js, fn, workers)


def hvp_sum(plan, directions, js, phi0_fn, workers=1):
    """(per-slot HVP [n,16], counts) (objective.py:432-482).  The reference
    always evaluates the HVP with a dense plan (objective.py:786)."""
    js = np.asarray(js, np.int64)
    N, n = 2**plan.k, plan.n
    zm, zt = plan.zmats(directions)

    def fn(jj):
        phi = _c(phi0_fn(jj))
        psis = np.empty((n + 1, N), np.complex128)
        phis = np.empty((n + 1, N), np.complex128)
        vb, tb = np.empty(N, np.complex128), np.empty(N, np.complex128)
        oacc = np.zeros((n, 16), np.complex128)
        counts = np.zeros(5, np.int64)
        jj = np.ascontiguousarray(jj)
        _lib.or_hvp_chunk(ctypes.byref(plan._c), _ptr(zm), _ptr(zt), _ptr(jj), _I(len(jj)), _ptr(phi), _ptr(psis),
                          _ptr(phis), _ptr(vb), _ptr(tb), _ptr(oacc), _ptr(counts))
        return oacc, counts

    return _reduce(js, fn, workers)


def hessian_sum(plan, js, phi0_fn, classes=None, workers=1):
    """(value, per-slot D, blocks[R,A,A], routes_used, counts) (objective.py:340-423)."""
    js = np.asarray(js, np.int64)
    N, n = 2**plan.k, plan.n
    A = len(plan.support)
    csr = pair_csr(plan.targets, plan.logical, plan.nlog, classes)
    first, start, sec, mult, route, sym, flip = csr
    R = plan.nlog * (plan.nlog + 1) // 2

    def fn(jj):
        phi = _c(phi0_fn(jj))
        psis = np.empty((n + 1, N), np.complex128)
        phis = np.empty((n + 1, N), np.complex128)
        h1, h2 = np.empty((N, A), np.complex128), np.empty((N, A), np.complex128)
        dacc = np.zeros((n, 16), np.complex128)
        blocks = np.zeros((R, A, A), np.complex128)
        out_t = np.empty((A, A), np.complex128)
        counts = np.zeros(5, np.int64)
        v = np.zeros(1, np.complex128)
        jj = np.ascontiguousarray(jj)
        _lib.or_hessian_chunk(ctypes.byref(plan._c), _ptr(plan.hole_row), _ptr(plan.hole_col), _I(A), _ptr(first),
                              _I(len(first)), _ptr(start), _ptr(sec), _ptr(mult), _ptr(route), _ptr(sym), _ptr(flip),
                              _ptr(jj), _I(len(jj)), _ptr(phi), _ptr(psis), _ptr(phis), _ptr(h1), _ptr(h2),
                              _ptr(dacc), _ptr(blocks), _ptr(out_t), _ptr(counts), _ptr(v))
        return v[0], dacc, blocks, counts

    v, dacc, blocks, counts = _reduce(js, fn, workers)
    used = sorted(set(int(r) for r in route))
    keys = []
    for a in range(plan.nlog):
        for b in range(a, plan.nlog):
            r = a * plan.nlog - a * (a - 1) // 2 + (b - a)
            if r in used:
                keys.append((a, b, r))
    return v, dacc, {(a, b): blocks[r] for a, b, r in keys}, counts


def grad_hvp_reversible(plan, directions, j, phi0_row):
    """One summand j: (value, per-slot D [n,16], per-slot HVP [n,16]) of the
    reference recursions (objective.py:307-337, 432-482) run in the reversible
    3-vector schedule from the restated cores (oracle/gf_oracle.c
    or_grad_hvp_reversible) -- the large-k oracle;
    host-parallel over tuples, 4 scratch vectors instead of 2(n+1)."""
    N, n = 2**plan.k, plan.n
    zm, zt = plan.zmats(directions)
    phi = _c(phi0_row)
    if phi.shape != (N,):
        raise ValueError("phi0 row must have 2**k amplitudes")
    bufs = [np.empty(N, np.complex128) for _ in range(4)]
    dacc = np.zeros((n, 16), np.complex128)
    oacc = np.zeros((n, 16), np.complex128)
    v = np.zeros(1, np.complex128)
    _lib.or_grad_hvp_reversible(ctypes.byref(plan._c), _ptr(zm), _ptr(zt), _I(int(j)), _ptr(phi),
                                *[_ptr(b) for b in bufs], _ptr(dacc), _ptr(oacc), _ptr(v))
    return v[0], dacc, oacc


# ---------------------------------------------------------------- models / targets


def chain_bonds(L, offset, periodic):
    """models.py:94-119 (merged duplicate wrap bond at L=2)."""
    even, odd, seen = [], [], {}
    for j in range(L):
        if j == L - 1 and not periodic:
            break
        bond = (offset + j, offset + (j + 1) % L)
        key = (min(bond), max(bond))
        if key in seen:
            seen[key][1] += 1
            continue
        e = [bond, 1]
        seen[key] = e
        (even if j % 2 == 0 else odd).append(e)
    return [tuple(e) for e in even], [tuple(e) for e in odd]


def spinful_terms(L, J, U, periodic):
    """models.py:149-170 -> (terms [(a, b, coeff, is_hop)], groups [bonds])."""
    ue, uo = chain_bonds(L, 0, periodic)
    de, do = chain_bonds(L, L, periodic)
    terms, groups = [], []
    for merged in (ue + de, uo + do):
        if not merged:
            continue
        for bond, m in merged:
            terms.append((bond[0], bond[1], -J * m, True))
        groups.append([b for b, _ in merged])
    ib = [(j, j + L) for j in range(L)]
    for b in ib:
        terms.append((b[0], b[1], U, False))
    groups.append(ib)
    return terms, groups


def spinless_terms(L, J, U, periodic):
    """models.py:129-146."""
    even, odd = chain_bonds(L, 0, periodic)
    terms, groups = [], []
    for merged in (even, odd):
        if not merged:
            continue
        for bond, m in merged:
            terms.append((bond[0], bond[1], -J * m, True))
            terms.append((bond[0], bond[1], U * m, False))
        groups.append([b for b, _ in merged])
    return terms, groups


class HamiltonianApply:
    def __init__(self, k, terms):
        self.k = k
        t = np.array(terms, dtype=object)
        self.a = np.ascontiguousarray([int(x[0]) for x in terms], np.int64)
        self.b = np.ascontiguousarray([int(x[1]) for x in terms], np.int64)
        self.c = np.ascontiguousarray([float(x[2]) for x in terms], np.float64)
        self.h = np.ascontiguousarray([int(bool(x[3])) for x in terms], np.int32)
        del t

    def __call__(self, psi):
        psi = _c(psi)
        out = np.empty_like(psi)
        _lib.or_hamiltonian_apply(ctypes.c_int(self.k), _ptr(self.a), _ptr(self.b), _ptr(self.c), _ptr(self.h),
                                  _I(len(self.a)), _ptr(psi), _ptr(out))
        return out


def dense_target(k, terms, t):
    """exp(-i H t) densely (models.py:258-319); k <= 14."""
    import scipy.linalg

    if k > 14:
        raise ValueError("dense target capped at 14 qubits")
    H = HamiltonianApply(k, terms)
    N = 2**k
    h = np.empty((N, N), np.complex128)
    e = np.zeros(N, np.complex128)
    for j in range(N):
        e[j] = 1.0
        h[:, j] = H(e)
        e[j] = 0.0
    return scipy.linalg.expm(-1j * t * h)


def lanczos_expm(H, state, t, tol=1e-12, max_dim=96):
    """Restates KrylovOracle._expm_multiply (models.py:343-384)."""
    import scipy.linalg

    norm = np.linalg.norm(state)
    if norm == 0.0 or t == 0.0:
        return np.asarray(state, np.complex128)
    basis = [state / norm]
    alphas, betas = [], []
    prev = None
    for _ in range(1, min(max_dim, state.size) + 1):
        w = H(basis[-1])
        if len(basis) > 1:
            w = w - betas[-1] * basis[-2]
        alpha = float(np.real(np.vdot(basis[-1], w)))
        w = w - alpha * basis[-1]
        for u in basis:
            w = w - np.vdot(u, w) * u
        alphas.append(alpha)
        beta = float(np.linalg.norm(w))
        m = len(alphas)
        if m == 1:
            coeff = np.array([np.exp(-1j * t * alphas[0])])
        else:
            ev, V = scipy.linalg.eigh_tridiagonal(alphas, betas[: m - 1])
            coeff = V @ (np.exp(-1j * t * ev) * V[0].conj())
        approx = sum(c * u for c, u in zip(coeff, basis))
        resid = beta * abs(coeff[-1]) * abs(t)
        step = np.inf if prev is None else np.linalg.norm(approx - prev)
        if beta < 1e-14 or max(resid, step) < tol:
            return norm * approx
        prev = approx
        betas.append(beta)
        basis.append(w / beta)
    raise RuntimeError("Lanczos did not converge")


def dense_phi0(U):
    """phi0(j) = conj(U|j>) for a dense target (objective.py:561-565)."""
    Uc = np.ascontiguousarray(np.conj(U).T)
    return lambda jj: Uc[np.asarray(jj)]


def lanczos_phi0(k, terms, t):
    H = HamiltonianApply(k, terms)
    N = 2**k

    def fn(jj):
        out = np.empty((len(jj), N), np.complex128)
        for i, j in enumerate(jj):
            e = np.zeros(N, np.complex128)
            e[int(j)] = 1.0
            out[i] = np.conj(lanczos_expm(H, e, t))
        return out

    return fn


# ---------------------------------------------------------------- sector / fold


def sector_unrank(idx, sector=0):
    idx = np.ascontiguousarray(idx, np.int64)
    out = np.empty_like(idx)
    _lib.or_sector_unrank(_ptr(idx), _I(idx.size), ctypes.c_int(sector), _ptr(out))
    return out


def sector_rank(x):
    x = np.ascontiguousarray(x, np.int64)
    out = np.empty_like(x)
    _lib.or_sector_rank(_ptr(x), _I(x.size), _ptr(out))
    return out


def orbit_canon(x, L):
    x = np.ascontiguousarray(x, np.int64)
    rep, size = np.empty_like(x), np.empty_like(x)
    _lib.or_orbit_canon(_ptr(x), _I(x.size), ctypes.c_int(L), _ptr(rep), _ptr(size))
    return rep, size


def sector_orbit_reps(L, sector=0):
    """(compressed rep indices ascending, orbit sizes) of the parity sector."""
    M = 2 ** (2 * L - 1)
    cap = M
    reps = np.empty(cap, np.int64)
    w = np.empty(cap, np.int64)
    cnt = _lib.or_sector_orbit_reps(ctypes.c_int(L), ctypes.c_int(sector), _ptr(reps), _ptr(w), _I(cap))
    return reps[:cnt].copy(), w[:cnt].copy()


_lib.or_sector_orbit_reps.restype = ctypes.c_int64
