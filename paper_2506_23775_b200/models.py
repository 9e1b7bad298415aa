"""Fermi-Hubbard target Hamiltonians, Trotter circuits and GPU target oracles.

Host-side setup with the semantics of the reference ``gatefit.models``
(reference models.py:37-393): hard-core-boson qubit mapping (Jordan-Wigner
order, spin-up chain first, wrap strings dropped), Trotter groups, the
closed-form two-site Trotter gate, and target oracles providing
``U|psi>`` with ``U = exp(-i H t)``.

Oracles expose the reference duck type (``num_qubits``, ``apply``,
``apply_adjoint``) and additionally ``phi0_into(js_full, sector, out)`` which
writes conj(U|j>) for a batch of basis states straight into device memory for
the engine:

* ``DenseOracle`` -- dense expm (k <= 14, reference models.py:305-319) kept on
  the GPU;
* ``ChebyshevOracle`` -- matrix-free exp(-iHt) on the GPU (Chebyshev
  expansion with a fused H-apply kernel); replaces the
  reference's CPU Lanczos ``KrylovOracle`` (models.py:322-384), which is kept
  as an alias name for drop-in use.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .circuit import BrickwallMeta, Circuit, GateSlot
from .kernels import Gate
from .manifold import parity_join, random_unitary

__all__ = [
    "Term",
    "TrotterGroup",
    "HamiltonianSpec",
    "TrotterPlan",
    "build_spinless_fh",
    "build_spinful_fh",
    "trotter_gate",
    "build_trotter_circuit",
    "hamiltonian_apply",
    "dense_hamiltonian",
    "make_oracle",
    "DenseOracle",
    "ChebyshevOracle",
    "NumberBlockOracle",
    "KrylovOracle",
    "KrylovConvergenceError",
    "spinful_layer_circuit",
    "CachedTargetColumns",
]

_HOP = np.array([[0, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 0]], dtype=np.complex128)
_NN = np.diag([0.0, 0.0, 0.0, 1.0]).astype(np.complex128)
_OPERATORS = {"hop": _HOP, "nn": _NN}


@dataclass(frozen=True)
class Term:
    coefficient: float
    operator: str
    sites: tuple[int, int]


@dataclass(frozen=True)
class TrotterGroup:
    bonds: tuple[tuple[int, int], ...]
    hop_coeff: float
    int_coeff: float


@dataclass
class HamiltonianSpec:
    num_qubits: int
    terms: list[Term]
    trotter_groups: list[TrotterGroup]
    brickwall: bool = False
    periodic: bool = False

    def __post_init__(self):
        for t in self.terms:
            a, b = t.sites
            if a == b or min(a, b) < 0 or max(a, b) >= self.num_qubits:
                raise ValueError(f"invalid term sites {t.sites}")
            if t.operator not in _OPERATORS:
                raise ValueError(f"unknown operator {t.operator!r}")

    def term_arrays(self):
        ta = np.array([t.sites[0] for t in self.terms], dtype=np.int32)
        tb = np.array([t.sites[1] for t in self.terms], dtype=np.int32)
        c = np.array([t.coefficient for t in self.terms], dtype=np.float64)
        h = np.array([t.operator == "hop" for t in self.terms], dtype=np.int32)
        return ta, tb, c, h

    def spectral_bounds(self):
        """Gershgorin interval containing the spectrum."""
        _, _, c, h = self.term_arrays()
        hop = np.abs(c[h == 1]).sum()
        nn = c[h == 0]
        lo = np.minimum(nn, 0).sum() - hop
        hi = np.maximum(nn, 0).sum() + hop
        return float(lo), float(hi)


@dataclass(frozen=True)
class TrotterPlan:
    order: int
    steps: int
    total_time: float

    def __post_init__(self):
        if self.order not in (1, 2, 4):
            raise ValueError(f"unsupported Trotter order {self.order}")
        if self.steps < 1:
            raise ValueError("steps must be >= 1")


def _chain(L: int, offset: int, periodic: bool):
    """Bonds of one chain split by bond parity, duplicate wrap bond (L=2)
    merged into multiplicity 2 (reference models.py:94-119)."""
    by_key: dict[tuple[int, int], list] = {}
    groups: tuple[list, list] = ([], [])
    last = L if periodic else L - 1
    for j in range(last):
        bond = (offset + j, offset + (j + 1) % L)
        key = tuple(sorted(bond))
        if key in by_key:
            by_key[key][1] += 1
        else:
            entry = [bond, 1]
            by_key[key] = entry
            groups[j % 2].append(entry)
    return [tuple(e) for e in groups[0]], [tuple(e) for e in groups[1]]


def _single_mult(entries):
    mults = {m for _, m in entries}
    if len(mults) != 1:
        raise AssertionError("mixed bond multiplicities within one Trotter group")
    return mults.pop()


def build_spinless_fh(L: int, J: float, U: float, periodic: bool = False) -> HamiltonianSpec:
    """-J sum hop + U sum n n on L qubits (reference models.py:129-146)."""
    if L < 2:
        raise ValueError("need at least two sites")
    terms, groups = [], []
    for entries in _chain(L, 0, periodic):
        if not entries:
            continue
        m = _single_mult(entries)
        for bond, mb in entries:
            terms += [Term(-J * mb, "hop", bond), Term(U * mb, "nn", bond)]
        groups.append(TrotterGroup(tuple(b for b, _ in entries), J * m, U * m))
    return HamiltonianSpec(L, terms, groups, brickwall=True, periodic=periodic)


def build_spinful_fh(L: int, J: float, U: float, periodic: bool = False) -> HamiltonianSpec:
    """2L qubits, up chain then down chain; on-site (j, j+L) interaction
    (reference models.py:149-170)."""
    if L < 2:
        raise ValueError("need at least two sites")
    up = _chain(L, 0, periodic)
    dn = _chain(L, L, periodic)
    terms, groups = [], []
    for entries in (up[0] + dn[0], up[1] + dn[1]):
        if not entries:
            continue
        m = _single_mult(entries)
        terms += [Term(-J * mb, "hop", bond) for bond, mb in entries]
        groups.append(TrotterGroup(tuple(b for b, _ in entries), J * m, 0.0))
    onsite = tuple((j, j + L) for j in range(L))
    terms += [Term(U, "nn", b) for b in onsite]
    groups.append(TrotterGroup(onsite, 0.0, U))
    return HamiltonianSpec(2 * L, terms, groups, brickwall=False, periodic=periodic)


def trotter_gate(J: float, U: float, t: float) -> Gate:
    """exp(-i t (-J hop + U nn)) in closed form (reference models.py:173-188)."""
    m = np.zeros((4, 4), dtype=np.complex128)
    c, s = np.cos(J * t), np.sin(J * t)
    m[0, 0] = 1.0
    m[1, 1] = m[2, 2] = c
    m[1, 2] = m[2, 1] = 1j * s
    m[3, 3] = np.exp(-1j * U * t)
    return Gate(m, (0, 1), parity_sparse=True)


def _strang(ng: int, tau: float):
    half = [(g, tau / 2.0) for g in range(ng - 1)]
    return half + [(ng - 1, tau)] + half[::-1]


def _layers(ng: int, order: int, steps: int, total: float):
    dt = total / steps
    if order == 1:
        step = [(g, dt) for g in range(ng)]
    elif order == 2:
        step = _strang(ng, dt)
    else:  # Suzuki fourth order from five Strang steps
        u = 1.0 / (4.0 - 4.0 ** (1.0 / 3.0))
        step = [x for c in (u, u, 1.0 - 4.0 * u, u, u) for x in _strang(ng, c * dt)]
    out: list[tuple[int, float]] = []
    for g, tt in step * steps:
        if out and out[-1][0] == g:
            out[-1] = (g, out[-1][1] + tt)
        else:
            out.append((g, tt))
    return out


def build_trotter_circuit(spec: HamiltonianSpec, plan: TrotterPlan) -> Circuit:
    """Trotterised exp(-iHt); one shared logical gate per merged layer
    (reference models.py:217-244)."""
    if not spec.trotter_groups:
        raise ValueError("hamiltonian spec has no Trotter bond groups")
    layers = _layers(len(spec.trotter_groups), plan.order, plan.steps, plan.total_time)
    gates, slots, layer_of = [], [], []
    for li, (g, tt) in enumerate(layers):
        grp = spec.trotter_groups[g]
        gates.append(Gate(trotter_gate(grp.hop_coeff, grp.int_coeff, tt).matrix, grp.bonds[0], parity_sparse=True))
        for bond in grp.bonds:
            slots.append(GateSlot(li, bond))
            layer_of.append(li)
    meta = None
    if spec.brickwall and all(g == i % 2 for i, (g, _) in enumerate(layers)):
        meta = BrickwallMeta(len(layers), tuple(layer_of), 2, spec.periodic)
    return Circuit(spec.num_qubits, slots, gates, meta)


def spinful_layer_circuit(L: int, num_layers: int, periodic: bool, seed: int, parity: bool = False,
                          J: float = 1.0, U: float = 4.0):
    """BASELINE.json config recipe: layer i uses Trotter
    group i mod 3 with one Haar-random logical gate (U(4), or U(2)xU(2) via
    parity_join(odd, even) when ``parity``) from ``default_rng(seed)``.
    Returns (spec, circuit, rng) -- the rng continues for tangent draws."""
    spec = build_spinful_fh(L, J, U, periodic)
    rng = np.random.default_rng(seed)
    slots, gates = [], []
    for layer in range(num_layers):
        grp = spec.trotter_groups[layer % len(spec.trotter_groups)]
        if parity:
            m = parity_join(random_unitary(2, rng), random_unitary(2, rng))
        else:
            m = random_unitary(4, rng)
        gates.append(Gate(m, grp.bonds[0], parity_sparse=parity))
        slots += [GateSlot(layer, b) for b in grp.bonds]
    return spec, Circuit(spec.num_qubits, slots, gates), rng


# ---------------------------------------------------------------- H apply


def _dense_embed(mat: np.ndarray, a: int, b: int, k: int) -> np.ndarray:
    """Dense 2^k x 2^k operator of a two-site matrix (qubit 0 = MSB)."""
    N = 1 << k
    x = np.arange(N)
    ba = (x >> (k - 1 - a)) & 1
    bb = (x >> (k - 1 - b)) & 1
    env = x & ~((1 << (k - 1 - a)) | (1 << (k - 1 - b)))
    out = np.zeros((N, N), dtype=np.complex128)
    for i in range(4):
        for j in range(4):
            if mat[i, j] == 0:
                continue
            rows = np.nonzero((2 * ba + bb) == i)[0]
            cols = env[rows] | ((j >> 1) << (k - 1 - a)) | ((j & 1) << (k - 1 - b))
            out[rows, cols] += mat[i, j]
    return out


def dense_hamiltonian(spec: HamiltonianSpec) -> np.ndarray:
    if spec.num_qubits > 14:
        raise ValueError("dense assembly capped at 14 qubits")
    N = 1 << spec.num_qubits
    h = np.zeros((N, N), dtype=np.complex128)
    for t in spec.terms:
        h += t.coefficient * _dense_embed(_OPERATORS[t.operator], t.sites[0], t.sites[1], spec.num_qubits)
    return h


def hamiltonian_apply(spec: HamiltonianSpec, state):
    """H|psi> matrix-free on the GPU (reference models.py:247-255)."""
    from .kernels import _finish, _stage

    s, host = _stage(state, 1)
    if s.shape[0] != 1 << spec.num_qubits:
        raise ValueError("state dimension does not match the Hamiltonian")
    out = torch.empty_like(s)
    ta, tb, c, h = spec.term_arrays()
    _lib.check(_lib.lib.gf_hamiltonian_apply(s.data_ptr(), out.data_ptr(), spec.num_qubits, ta.ctypes.data,
                                             tb.ctypes.data, c.ctypes.data, h.ctypes.data, len(ta), 1,
                                             _lib.stream_ptr()))
    return _finish(out, host)


# ---------------------------------------------------------------- oracles


class KrylovConvergenceError(RuntimeError):
    """Kept for API parity with the reference (models.py:301-302)."""


def _unrank_host(i: np.ndarray, sector: int) -> np.ndarray:
    pc = np.array([bin(int(v)).count("1") & 1 for v in np.atleast_1d(i)], dtype=np.int64)
    return (np.asarray(i, np.int64) << 1) | (pc ^ sector)


class DenseOracle:
    """exp(-iHt) formed densely on the host (k <= 14) and kept on the GPU."""

    def __init__(self, spec: HamiltonianSpec, t: float):
        import scipy.linalg

        if spec.num_qubits > 14:
            raise ValueError("dense oracle capped at 14 qubits")
        self.num_qubits = spec.num_qubits
        self.spec = spec
        self._u = scipy.linalg.expm(-1j * t * dense_hamiltonian(spec))
        self._cols = None
        self._sector_cols = {}

    @classmethod
    def from_matrix(cls, u: np.ndarray):
        o = cls.__new__(cls)
        o.num_qubits = int(u.shape[0]).bit_length() - 1
        o._u = np.ascontiguousarray(u, dtype=np.complex128)
        o._cols = None
        o._sector_cols = {}
        return o

    def apply(self, state):
        return self._u @ state

    def apply_adjoint(self, state):
        return np.conj(self._u).T @ state

    def _device_cols(self, device):
        if self._cols is None or self._cols.device != device:
            # row j = conj(U[:, j]) = phi0 of basis state j
            self._cols = torch.from_numpy(np.ascontiguousarray(np.conj(self._u).T)).to(device)
        return self._cols

    def phi0_into(self, js_full: torch.Tensor, sector, out: torch.Tensor) -> None:
        cols = self._device_cols(out.device)
        if sector is None:
            torch.index_select(cols, 0, js_full, out=out)
            return
        if sector not in self._sector_cols:
            full = _unrank_host(np.arange(1 << (self.num_qubits - 1)), sector)
            self._sector_cols[sector] = torch.from_numpy(full).to(out.device)
        rows = torch.index_select(cols, 0, js_full)
        torch.index_select(rows, 1, self._sector_cols[sector], out=out)


class ChebyshevOracle:
    """Matrix-free exp(-iHt)|j> on the GPU by a Chebyshev expansion.

    H~ = (H - a)/b maps the Gershgorin interval onto [-1, 1];
    exp(-iHt) = e^{-iat} [J_0(bt) + 2 sum_m (-i)^m J_m(bt) T_m(H~)].  Since H and
    |j> are real, phi0 = conj(U|j>) = sum conj(c_m) T_m(H~)|j>.  Terms stop
    when |J_m(bt)| < tol.  Works in the compressed parity sector directly.
    """

    def __init__(self, spec: HamiltonianSpec, t: float, tol: float = 1e-16, max_batch: int | None = None):
        from scipy.special import jv

        self.num_qubits = spec.num_qubits
        self.spec = spec
        self.t = float(t)
        lo, hi = spec.spectral_bounds()
        self.a = 0.5 * (hi + lo)
        self.b = 0.5 * (hi - lo) * 1.01 + 1e-12
        bt = self.b * self.t
        M = int(abs(bt)) + 8
        while abs(jv(M, bt)) > tol or M < abs(bt):
            M += 1
        m = np.arange(M + 1)
        c = jv(m, bt) * (-1j) ** m * 2.0
        c[0] /= 2.0
        c *= np.exp(-1j * self.a * self.t)
        self.coef = np.conj(c)  # coefficients of conj(U|j>)
        self.order = M
        self._terms = spec.term_arrays()
        self.max_batch = max_batch

    # reference duck type (host vectors; used by generic code paths)
    def apply(self, state):
        return self._expm_host(np.asarray(state, np.complex128), self.t)

    def apply_adjoint(self, state):
        return self._expm_host(np.asarray(state, np.complex128), -self.t)

    def _expm_host(self, state, t):
        o = self if t == self.t else ChebyshevOracle(self.spec, t)
        dev = torch.device("cuda", torch.cuda.current_device())
        re = torch.from_numpy(np.ascontiguousarray(state.real)).to(dev, torch.complex128)
        im = torch.from_numpy(np.ascontiguousarray(state.imag)).to(dev, torch.complex128)
        # U(re + i im) = U re + i U im with real inputs: conj(o.series(x)) = U x
        ur = torch.conj(o._series(re[None], None))[0]
        ui = torch.conj(o._series(im[None], None))[0]
        return (ur + 1j * ui).cpu().numpy()

    def _series(self, v0: torch.Tensor, sector, out: torch.Tensor | None = None) -> torch.Tensor:
        """sum conj(c_m) T_m(H~) v0 for a real-valued batch v0 [B, N]."""
        B, N = v0.shape
        ta, tb, c, h = self._terms
        flags = 3 if sector is None else int(sector)
        acc = out if out is not None else torch.empty_like(v0)
        acc.copy_(v0 * complex(self.coef[0]))
        prev, cur = None, v0
        nxt = torch.empty_like(v0)
        spare = torch.empty_like(v0)
        scale, shift = 1.0 / self.b, -self.a / self.b
        st = _lib.stream_ptr()
        for m in range(1, self.order + 1):
            cm = complex(self.coef[m])
            _lib.check(_lib.lib.gf_cheb_step(cur.data_ptr(), None if prev is None else prev.data_ptr(),
                                             nxt.data_ptr(), acc.data_ptr(), self.num_qubits, ta.ctypes.data,
                                             tb.ctypes.data, c.ctypes.data, h.ctypes.data, len(ta), scale, shift,
                                             cm.real, cm.imag, B, flags, st))
            if prev is None:
                prev, cur, nxt = cur, nxt, spare
            else:
                prev, cur, nxt = cur, nxt, prev
        return acc

    def phi0_into(self, js_full: torch.Tensor, sector, out: torch.Tensor) -> None:
        B, N = out.shape
        v0 = torch.zeros_like(out)
        idx = js_full if sector is None else (js_full >> 1)
        v0[torch.arange(B, device=out.device), idx] = 1.0
        self._series(v0, sector, out=out)


_NB_INDEX_MAPS: dict = {}


class NumberBlockOracle(ChebyshevOracle):
    """exp(-iHt)|j> inside j's particle-number block, on the GPU.

    Hopping terms conserve the occupation of each connected component of the
    hop graph (each spin chain of the Fermi-Hubbard models, reference
    models.py:37-45, 247-255), so U|j> is supported on the states with j's
    particle count per component: C(8,a) C(8,b) <= 4900 of 65536 states at
    16 qubits.  The same Chebyshev series as :class:`ChebyshevOracle` runs in
    block coordinates (colex ranks, csrc/gf_target.cu), then the block
    vectors are scattered into dense (or sector-compressed) rows.  Blocks of
    dimension <= ``cache_dim`` are expanded once as whole matrices (the
    series on the identity) and reused for every column of the block; larger
    blocks run the series on the requested columns only.
    """

    def __init__(self, spec: HamiltonianSpec, t: float, tol: float = 1e-16, cache_dim: int = 8192):
        super().__init__(spec, t, tol)
        k = spec.num_qubits
        ta, tb, c, h = self._terms
        parent = list(range(k))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a

        for a, b, hop in zip(ta, tb, h):
            if hop:
                parent[find(int(a))] = find(int(b))
        comps = {}
        for q in range(k):
            comps.setdefault(find(q), []).append(q)
        self.components = sorted(comps.values())
        if len(self.components) > 4 or max(len(cq) for cq in self.components) > 32:
            raise ValueError("number-block oracle supports <= 4 hop components of <= 32 qubits")
        where = {}
        for ci, cq in enumerate(self.components):
            for i, q in enumerate(cq):
                where[q] = (ci, i)
        rows = []
        for a, b, hop in zip(ta, tb, h):
            ca, ia = where[int(a)]
            cb, ib = where[int(b)]
            rows.append((0 if hop else 1, ca, ia, cb, ib))
        self._nb_terms = np.ascontiguousarray(np.array(rows, np.int32).reshape(-1, 5))
        self._nb_coef = np.ascontiguousarray(c, np.float64)
        self._masks = np.array([sum(1 << (k - 1 - q) for q in cq) for cq in self.components], np.int64)
        self.cache_dim = int(cache_dim)
        self._blocks = {}
        self._tab = None

    def block_of(self, j: int):
        return tuple(bin(int(j) & int(m)).count("1") for m in self._masks)

    def block_dim(self, counts) -> int:
        from math import comb

        d = 1
        for cq, n in zip(self.components, counts):
            d *= comb(len(cq), n)
        return d

    def _desc(self, counts):
        d = [self.num_qubits, len(self.components)]
        for cq, n in zip(self.components, counts):
            d += [len(cq), int(n)] + list(cq)
        return np.ascontiguousarray(np.array(d, np.int32))

    def _block_series(self, desc, v0: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """sum conj(c_m) T_m(H~) v0 for block vectors v0 [B, D]."""
        B = v0.shape[0]
        acc = out if out is not None else torch.empty_like(v0)
        torch.mul(v0, complex(self.coef[0]), out=acc)
        prev, cur = None, v0
        nxt = torch.empty_like(v0)
        spare = torch.empty_like(v0)
        scale, shift = 1.0 / self.b, -self.a / self.b
        st = _lib.stream_ptr()
        tr, co = self._nb_terms, self._nb_coef
        for m in range(1, self.order + 1):
            cm = complex(self.coef[m])
            _lib.check(_lib.lib.gf_nb_cheb_step(cur.data_ptr(), None if prev is None else prev.data_ptr(),
                                                nxt.data_ptr(), acc.data_ptr(), desc.ctypes.data, len(desc),
                                                tr.ctypes.data, co.ctypes.data, len(co), scale, shift, cm.real,
                                                cm.imag, B, st))
            if prev is None:
                prev, cur, nxt = cur, nxt, spare
            else:
                prev, cur, nxt = cur, nxt, prev
        return acc

    def _ranks(self, desc, js: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(js)
        _lib.check(_lib.lib.gf_nb_rank(js.data_ptr(), out.data_ptr(), js.numel(), desc.ctypes.data, len(desc),
                                       _lib.stream_ptr()))
        return out

    def block_matrix(self, counts) -> torch.Tensor:
        """[D, D] rows = conj(U e_x) in block coordinates (cached)."""
        counts = tuple(int(n) for n in counts)
        mat = self._blocks.get(counts)
        if mat is None:
            D = self.block_dim(counts)
            dev = torch.device("cuda", torch.cuda.current_device())
            mat = self._block_series(self._desc(counts), torch.eye(D, dtype=torch.complex128, device=dev))
            self._blocks[counts] = mat
        return mat

    def _tables(self):
        """Whole-space block tables (when every block has dimension <=
        cache_dim): every block matrix in one device buffer plus the maps
        state -> (block, rank) and (block, rank) -> state, so target rows are
        gathered on the device without a host round trip."""
        if self._tab is not None:
            return self._tab or None
        from math import comb

        k = self.num_qubits
        largest = 1
        for cq in self.components:
            largest *= comb(len(cq), len(cq) // 2)
        if k > 26 or largest > self.cache_dim:
            self._tab = False
            return None
        dev = torch.device("cuda", torch.cuda.current_device())
        idx = self._index_maps(dev)
        keys, dims, matoff = idx["keys"], idx["dims"], idx["matoff"]
        mats = torch.empty(int((dims * dims).sum()), dtype=torch.complex128, device=dev)
        coefs = torch.from_numpy(np.ascontiguousarray(self.coef, np.complex128)).to(dev)
        nh = max(1, int(self._nb_terms[:, 0].tolist().count(0)))
        work = torch.empty(int(dims.max()) * (16 + 12 * nh) // 8 + 1, dtype=torch.float64, device=dev)
        st = _lib.stream_ptr()
        tr, co = self._nb_terms, self._nb_coef
        for bi, counts in enumerate(keys):
            D = int(dims[bi])
            dst = mats[matoff[bi]:matoff[bi] + D * D].view(D, D)
            desc = self._desc(counts)
            if D <= 6400:  # whole series on chip, one launch per block
                _lib.check(_lib.lib.gf_nb_block_matrix(dst.data_ptr(), desc.ctypes.data, len(desc), tr.ctypes.data,
                                                       co.ctypes.data, len(co), coefs.data_ptr(), self.order,
                                                       1.0 / self.b, -self.a / self.b, work.data_ptr(), st))
            else:
                self._block_series(desc, torch.eye(D, dtype=torch.complex128, device=dev), out=dst)
        self._tab = dict(idx["dev"], mats=mats, max_dim=int(dims.max()))
        return self._tab

    def _index_maps(self, dev):
        """state <-> (block, rank) maps of the whole space.  They depend only
        on the hop graph (not on t or the coefficients), so they are shared by
        every oracle of the same structure."""
        from math import comb

        key = (self.num_qubits, tuple(tuple(c) for c in self.components), str(dev))
        hit = _NB_INDEX_MAPS.get(key)
        if hit is not None:
            return hit
        k = self.num_qubits
        states = np.arange(1 << k, dtype=np.int64)
        occ = np.stack([np.bitwise_count(states & m).astype(np.int64) for m in self._masks], axis=1)
        keys, block_of = np.unique(occ, axis=0, return_inverse=True)
        block_of = block_of.reshape(-1)
        dims = np.array([self.block_dim(c) for c in keys], dtype=np.int64)
        binom = np.array([[comb(a, b) for b in range(34)] for a in range(33)], dtype=np.int64)
        rank = np.zeros(1 << k, dtype=np.int64)
        stride = np.ones(1 << k, dtype=np.int64)
        for ci, cq in enumerate(self.components):
            cnt = np.zeros(1 << k, dtype=np.int64)
            r = np.zeros(1 << k, dtype=np.int64)
            for i, q in enumerate(cq):
                bit = (states >> (k - 1 - q)) & 1
                r += bit * binom[i, cnt + 1]
                cnt += bit
            rank += r * stride
            stride *= binom[len(cq), occ[:, ci]]
        full_of = np.lexsort((rank, block_of)).astype(np.int64)
        stoff = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
        matoff = np.concatenate([[0], np.cumsum(dims * dims)[:-1]]).astype(np.int64)
        put = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a.astype(dt))).to(dev)
        hit = {"keys": keys, "dims": dims, "matoff": matoff,
               "dev": {"matoff": put(matoff, np.int64), "stoff": put(stoff, np.int64), "blkdim": put(dims, np.int32),
                       "block_of": put(block_of, np.int32), "rank_of": put(rank, np.int32),
                       "full_of": put(full_of, np.int64)}}
        _NB_INDEX_MAPS[key] = hit
        return hit

    def phi0_into(self, js_full: torch.Tensor, sector, out: torch.Tensor) -> None:
        B, N = out.shape
        out.zero_()
        tab = self._tables()
        if tab is not None:
            js = js_full.contiguous()
            st = _lib.stream_ptr()
            for r0 in range(0, B, 65535):
                nr = min(B, r0 + 65535) - r0
                _lib.check(_lib.lib.gf_nb_gather(
                    js[r0:].data_ptr(), nr, tab["mats"].data_ptr(), tab["matoff"].data_ptr(),
                    tab["stoff"].data_ptr(), tab["blkdim"].data_ptr(), tab["block_of"].data_ptr(),
                    tab["rank_of"].data_ptr(), tab["full_of"].data_ptr(), tab["max_dim"],
                    0 if sector is None else 1, out[r0:].data_ptr(), N, st))
            return
        js_host = js_full.cpu().numpy().astype(np.int64)
        occ = np.stack([np.bitwise_count(js_host & m) for m in self._masks], axis=1)
        keys, inv = np.unique(occ, axis=0, return_inverse=True)
        sec = -1 if sector is None else int(sector)
        st = _lib.stream_ptr()
        dev = out.device
        for bi, counts in enumerate(keys):
            sel = np.nonzero(inv.reshape(-1) == bi)[0]
            desc = self._desc(counts)
            rows = torch.from_numpy(sel).to(dev)
            cols = self._ranks(desc, js_full[rows].contiguous())
            D = self.block_dim(counts)
            if D <= self.cache_dim:
                src = self.block_matrix(counts)
            else:
                v0 = torch.zeros((len(sel), D), dtype=torch.complex128, device=dev)
                v0[torch.arange(len(sel), device=dev), cols] = 1.0
                src = self._block_series(desc, v0)
                cols = None
            _lib.check(_lib.lib.gf_nb_scatter(src.data_ptr(), None if cols is None else cols.data_ptr(),
                                              out.data_ptr(), rows.data_ptr(), len(sel), N, desc.ctypes.data,
                                              len(desc), sec, st))


class CachedTargetColumns:
    """phi0 rows for basis positions [p0, p1) of one basis-sum layout,
    computed once by an inner oracle and kept resident in HBM (the target
    does not change across trust-region iterations).  ``phi0_at`` hands the
    engine zero-copy views; positions outside the cached range fall back to
    the inner oracle."""

    def __init__(self, oracle, k: int, p0: int, p1: int, sector=None, indices=None, batch: int = 256):
        self.num_qubits = oracle.num_qubits
        self.inner = oracle
        self.spec = getattr(oracle, "spec", None)
        self.p0, self.p1 = p0, p1
        self.sector = sector
        self.indices = None if indices is None else np.asarray(indices, np.int64).copy()
        dev = torch.device("cuda", torch.cuda.current_device())
        N = 1 << (k - (0 if sector is None else 1))
        self.rows = torch.empty((p1 - p0, N), dtype=torch.complex128, device=dev)
        for s in range(p0, p1, batch):
            e = min(p1, s + batch)
            if indices is None:
                st = torch.arange(s, e, dtype=torch.int64, device=dev)
            else:
                st = torch.from_numpy(np.ascontiguousarray(indices[s:e])).to(dev)
            if sector is None:
                js = st
            else:
                js = torch.empty_like(st)
                _lib.check(_lib.lib.gf_sector_unrank(st.data_ptr(), st.numel(), int(sector), js.data_ptr(),
                                                     _lib.stream_ptr()))
            oracle.phi0_into(js, sector, self.rows[s - p0:e - p0])

    def apply(self, state):
        return self.inner.apply(state)

    def apply_adjoint(self, state):
        return self.inner.apply_adjoint(state)

    def phi0_into(self, js_full, sector, out):
        self.inner.phi0_into(js_full, sector, out)

    def phi0_at(self, pos: int, nvec: int, sector_code: int, indices=None):
        want = None if sector_code < 0 else sector_code
        if want != self.sector or pos < self.p0 or pos + nvec > self.p1:
            return None
        if (indices is None) != (self.indices is None):
            return None
        if indices is not None and not np.array_equal(indices[pos:pos + nvec],
                                                      self.indices[pos:pos + nvec]):
            return None
        return self.rows[pos - self.p0:pos - self.p0 + nvec]


#: drop-in name for the reference's matrix-free oracle (models.py:322)
KrylovOracle = ChebyshevOracle


def make_oracle(spec: HamiltonianSpec, t: float, method: str = "dense"):
    """Reference models.py:387-393; ``"krylov"`` / ``"chebyshev"`` select the
    matrix-free GPU oracle."""
    if method == "dense":
        return DenseOracle(spec, t)
    if method in ("krylov", "chebyshev"):
        return ChebyshevOracle(spec, t)
    if method == "blocks":
        return NumberBlockOracle(spec, t)
    raise ValueError(f"unknown oracle method {method!r}")
