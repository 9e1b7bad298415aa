"""Basis-sum objective, gradient, Hessian-vector product and Hessian on the GPU.

Drop-in for the public API of the reference ``gatefit.objective``
(reference objective.py:586-814): the same functions, arguments, return
types, orientation conventions and exceptions.  The per-summand passes and
the reduction over basis states run in libgfcuda.so (gf_plan_eval); this
module only plans batches, fetches target columns from the oracle, shards
chunks over ranks and converts holomorphic derivatives to Riemannian
gradients on the host.

f(G) = -Re Tr[U^dag C(G)] = -Re sum_j phi0_j . C|j>,  phi0_j = conj(U|j>)
(reference objective.py:1-10).  Extra keyword-only options (no reference
counterpart):

* ``sector`` -- None (reference semantics), "even"/"odd" or 0/1: restrict the
  basis sum to a parity sector and store vectors compressed on qubit k-1
  (gates touching it become parity-controlled one-qubit gates);
* ``fold`` -- with a sector, sum over lattice-translation orbit
  representatives weighted by orbit size (periodic, translation-invariant
  circuit and target only);
* ``basis`` -- explicit ``(indices, weights)`` sample of stored-space indices;
* ``batch`` / ``chunk`` -- summands per engine call / per output record.

Reductions are deterministic: every summand is reduced by a fixed CTA tree,
chunks of ``chunk`` consecutive summands form records, and records are
summed in ascending chunk order -- bit-identical for any batch size and any
number of GPUs (the reference's worker-count invariance,
objective.py:490-533).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, manifold
from .circuit import Circuit, accumulate_shared, translation_classes
from .kernels import DENSE_SUPPORT, PARITY_SUPPORT, WIRE_SWAP, Gate, apply_gate, basis_state, hole_contract

__all__ = [
    "PassCache",
    "HessianBlocks",
    "ObjectiveReport",
    "target_value",
    "summand_gradient",
    "full_gradient",
    "gradient_and_hvp",
    "full_hessian",
    "hessian_vector_product",
    "hessian_vector_products",
    "build_pass_cache",
    "parallel_reduce",
    "chunk_bounds",
    "frobenius_error_squared",
    "default_workers",
    "BasisSpec",
    "check_translation_invariant",
]

COUNT_NAMES = (
    "gate_applications",
    "array_gate_applications",
    "hole_applications",
    "hole_contractions",
    "pair_contractions",
)
CHUNK_STATES = 64  # reference objective.py:75


def default_workers() -> int:
    """RQCO_WORKERS (reference objective.py:78-83); accepted for API parity --
    the GPU engine does not use host worker threads."""
    try:
        return max(1, int(os.environ.get("RQCO_WORKERS", "1")))
    except ValueError:
        return 1


@dataclass
class PassCache:
    forward_states: list
    backward_states: list


@dataclass
class HessianBlocks:
    """Upper-triangular holomorphic second-derivative blocks keyed (a, b),
    a <= b, over ``support`` entries (reference objective.py:99-131)."""

    num_logical: int
    support: np.ndarray
    blocks: dict

    def apply_direction(self, directions):
        if len(directions) != self.num_logical:
            raise ValueError("need one direction matrix per logical gate")
        sup = np.asarray(self.support)
        z = [np.asarray(d, dtype=np.complex128).reshape(16)[sup] for d in directions]
        acc = [np.zeros(sup.size, dtype=np.complex128) for _ in range(self.num_logical)]
        for (a, b), blk in self.blocks.items():
            acc[a] += blk @ z[b]
            if a != b:
                acc[b] += blk.T @ z[a]
        out = []
        for v in acc:
            m = np.zeros(16, dtype=np.complex128)
            m[sup] = v
            out.append(m.reshape(4, 4))
        return out


@dataclass
class ObjectiveReport:
    value: float
    per_logical_gradient: list | None = None
    euclidean_gradients: list | None = None
    holomorphic_derivatives: list | None = None
    hessian: HessianBlocks | None = None
    wall_time: float = 0.0
    pass_counts: dict = field(default_factory=dict)
    engine: dict = field(default_factory=dict)


def frobenius_error_squared(value: float, num_qubits: int) -> float:
    """||C - U||_F^2 = 2 Tr[I] + 2 f (reference objective.py:147-149)."""
    return 2.0 * 2**num_qubits + 2.0 * value


def chunk_bounds(total: int, num_chunks: int | None = None):
    """Contiguous near-equal chunks covering range(total) (reference
    objective.py:490-510)."""
    if total < 0:
        raise ValueError("total must be non-negative")
    if total == 0:
        return []
    nc = max(1, total // CHUNK_STATES) if num_chunks is None else num_chunks
    nc = max(1, min(nc, total))
    q, r = divmod(total, nc)
    edges = np.cumsum([0] + [q + (1 if c < r else 0) for c in range(nc)])
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


def parallel_reduce(num_items: int, evaluate_chunk, worker_count: int = 1):
    """Fixed chunks, partials combined with + in ascending order (reference
    objective.py:513-533).  Host helper kept for API parity."""
    if worker_count < 1:
        raise ValueError("worker_count must be >= 1")
    bounds = chunk_bounds(num_items)
    if not bounds:
        return None
    if worker_count == 1:
        parts = [evaluate_chunk(a, b) for a, b in bounds]
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=worker_count) as ex:
            parts = list(ex.map(lambda ab: evaluate_chunk(*ab), bounds))
    total = parts[0]
    for p in parts[1:]:
        total = total + p
    return total


# ---------------------------------------------------------------------------
# engine plan (C ABI) and basis planning
# ---------------------------------------------------------------------------


def _sector_code(sector) -> int:
    if sector is None:
        return -1
    if sector in ("even", 0):
        return 0
    if sector in ("odd", 1):
        return 1
    raise ValueError(f"unknown sector {sector!r}")


class EnginePlan:
    """Owns one gf_plan (device workspace for `batch` summands)."""

    def __init__(self, circuit: Circuit, sector: int, batch: int, chunk: int):
        t1, t2, lid = circuit.slot_arrays()
        self.k = circuit.num_qubits
        self.sector = sector
        self.batch = batch
        self.chunk = chunk
        self.nlog = circuit.num_logical
        self.n = circuit.num_slots
        self.N = 1 << (self.k - (1 if sector >= 0 else 0))
        self.rec = 2 + 64 * self.nlog
        self.nd = 1
        h = ctypes.c_void_p()
        self._keep = (t1, t2, lid)
        with torch.cuda.device(torch.cuda.current_device()):
            _lib.check(_lib.lib.gf_plan_create(ctypes.byref(h), self.k, sector, self.n, t1.ctypes.data,
                                               t2.ctypes.data, lid.ctypes.data, self.nlog, batch, chunk))
        self.h = h
        self.device = torch.device("cuda", torch.cuda.current_device())

    def set_gates(self, mats: np.ndarray):
        m = np.ascontiguousarray(mats, dtype=np.complex128)
        _lib.check(_lib.lib.gf_plan_set_gates(self.h, m.ctypes.data))

    def set_directions(self, zmats: np.ndarray):
        """[n_logical, 4, 4] (one direction) or [nd, n_logical, 4, 4] (nd <= 3
        directions evaluated in one set of sweeps)."""
        z = np.ascontiguousarray(zmats, dtype=np.complex128)
        nd = 1 if z.ndim == 3 else z.shape[0]
        _lib.check(_lib.lib.gf_plan_set_directions_multi(self.h, nd, z.ctypes.data))
        self.nd = nd
        self.rec = 2 + 32 * self.nlog * (1 + nd)

    def eval(self, flags, nvec, basis, weights, phi0, out):
        _lib.check(_lib.lib.gf_plan_eval(self.h, flags, nvec, basis.data_ptr(),
                                         None if weights is None else weights.data_ptr(), phi0.data_ptr(),
                                         out.data_ptr(), _lib.stream_ptr()))

    def slot_outputs(self, nvec: int):
        """Per-slot D and H sums (normalised wire orientation) of the last
        eval's batch: two complex arrays [n_slots, 4, 4]."""
        d = torch.empty((max(self.n, 1), 16), dtype=torch.complex128, device=self.device)
        h = torch.empty_like(d)
        _lib.check(_lib.lib.gf_plan_slot_outputs(self.h, nvec, d.data_ptr(), h.data_ptr(), _lib.stream_ptr()))
        return d[: self.n].reshape(-1, 4, 4).cpu().numpy(), h[: self.n].reshape(-1, 4, 4).cpu().numpy()

    def describe(self) -> dict:
        v = (ctypes.c_int * 5)()
        _lib.check(_lib.lib.gf_plan_describe(self.h, ctypes.byref(v, 0), ctypes.byref(v, 4), ctypes.byref(v, 8),
                                             ctypes.byref(v, 12), ctypes.byref(v, 16)))
        f = (ctypes.c_double * 3)()
        _lib.check(_lib.lib.gf_plan_live_fraction(self.h, f))
        return {"fused": bool(v[0]), "tile_bits": v[1], "fwd_passes": v[2], "rev_passes": v[3], "ctas": v[4],
                "live_fraction": {"forward": f[0], "reverse": f[1], "ascending": f[2]}}

    def last_launches(self) -> int:
        return int(_lib.lib.gf_plan_last_launches(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                _lib.lib.gf_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass


_PLANS: dict = {}
# environment knobs read by gf_plan_create (csrc/gf_engine.cu plan_knobs): part
# of the plan cache key so a changed knob never reuses a plan built without it
_PLAN_KNOBS = ("GF_ENGINE", "GF_FUSED_M", "GF_FWD_M", "GF_FUSED_C", "GF_FUSED_CTAS", "GF_PLAN_GREEDY",
               "GF_SPARSE_DMMA", "GF_C1Q_DMMA", "GF_PAIR_BLOCKS", "GF_SECTOR_FMA", "GF_UNIT_NT", "GF_LIGHTCONE", "GF_PLAN_MINPASS", "GF_PLAN_EXTRA")


def _get_plan(circuit: Circuit, sector: int, batch: int, chunk: int) -> EnginePlan:
    t1, t2, lid = circuit.slot_arrays()
    key = (torch.cuda.current_device(), circuit.num_qubits, sector, t1.tobytes(), t2.tobytes(), lid.tobytes(),
           circuit.num_logical, batch, chunk) + tuple(os.environ.get(v) for v in _PLAN_KNOBS)
    plan = _PLANS.get(key)
    if plan is None:
        while len(_PLANS) >= 4:
            _PLANS.pop(next(iter(_PLANS)))
        plan = EnginePlan(circuit, sector, batch, chunk)
        _PLANS[key] = plan
    return plan


@dataclass
class BasisSpec:
    """Summands of the basis sum in stored (possibly compressed) space.

    ``indices`` None means all stored indices 0..total-1 (contiguous)."""

    total: int
    indices: np.ndarray | None = None
    weights: np.ndarray | None = None

    def weight_sum(self) -> float:
        return float(self.total if self.weights is None else np.sum(self.weights))


def _default_batch(N: int, total: int) -> int:
    env = os.environ.get("GF_BATCH")
    if env:
        return max(1, min(int(env), total))
    # bytes per workspace vector (3 resident): batch 2048 at 16 qubits (measured at c2:
    # 50 355 / 51 250 / 51 827 / 51 860 summand-evals/s at batch 512 / 1024 / 2048 / 4096)
    budget = 2048 * 2**20
    return max(1, min(total, budget // (16 * N)))


def fold_basis(k: int, sector: int, L: int | None = None) -> BasisSpec:
    """Translation-orbit representatives of the sector with orbit sizes
    (computed on the GPU by gf_sector_orbit_mark)."""
    if sector < 0:
        raise ValueError("translation folding needs a parity sector")
    if L is None:
        if k % 2:
            raise ValueError("folding needs a spinful chain (even qubit count)")
        L = k // 2
    M = 1 << (k - 1)
    dev = torch.device("cuda", torch.cuda.current_device())
    reps, ws = [], []
    step = 1 << 26
    for i0 in range(0, M, step):
        m = min(step, M - i0)
        mark = torch.empty(m, dtype=torch.int32, device=dev)
        _lib.check(_lib.lib.gf_sector_orbit_mark(i0, m, L, sector, mark.data_ptr(), _lib.stream_ptr()))
        nz = torch.nonzero(mark).flatten()
        reps.append((nz + i0).cpu().numpy())
        ws.append(mark[nz].to(torch.float64).cpu().numpy())
    idx = np.concatenate(reps).astype(np.int64)
    return BasisSpec(int(idx.size), idx, np.concatenate(ws))


def _shift2(q: int, k: int) -> int:
    """Qubit image under the 2-site translation of both spin chains (qubit
    c*L + s -> c*L + (s + 2) mod L, L = k/2)."""
    L = k // 2
    c, s = divmod(q, L)
    return c * L + (s + 2) % L


def check_translation_invariant(circuit: Circuit, oracle=None):
    """Raise ValueError unless folding the basis sum by 2-site translations is
    exact: the circuit maps onto itself under the shift (every slot's image is
    a slot of the same logical gate with the same target order, and slots
    sharing a qubit keep their relative order) and, when the oracle exposes
    its Hamiltonian spec, the target is periodic and translation-invariant."""
    k = circuit.num_qubits
    if k % 2 or k < 4:
        raise ValueError("translation folding needs a spinful chain (even qubit count >= 4)")
    where = {}
    for i, s in enumerate(circuit.slots):
        where.setdefault((s.logical_id, s.targets), []).append(i)
    img = []
    for s in circuit.slots:
        key = (s.logical_id, (_shift2(s.targets[0], k), _shift2(s.targets[1], k)))
        cand = where.get(key)
        if not cand:
            raise ValueError(f"fold=True: the image of slot {s.targets} (logical {s.logical_id}) under the 2-site "
                             "translation is not a slot of the same logical gate; the circuit is not "
                             "translation-invariant (periodic, one gate per layer)")
        img.append(cand[0] if len(cand) == 1 else -1)
    if -1 in img:
        raise ValueError("fold=True: duplicate slots make the translation image ambiguous")
    n = circuit.num_slots
    qs = [set(s.targets) for s in circuit.slots]
    for a in range(n):
        for b in range(a + 1, n):
            if qs[a] & qs[b] and img[a] > img[b]:
                raise ValueError("fold=True: the 2-site translation reorders non-commuting slots")
    spec = getattr(oracle, "spec", None)
    if spec is not None:
        if not getattr(spec, "periodic", False):
            raise ValueError("fold=True needs a periodic (translation-invariant) target Hamiltonian")
        terms = {(t.operator, tuple(t.sites), float(t.coefficient)) for t in spec.terms}

        def canon(op, a, b):
            return (op, (a, b)) if op != "hop" else (op, (min(a, b), max(a, b)))

        tset = {canon(o, *st) + (c,) for o, st, c in terms}
        for o, st, c in terms:
            if canon(o, _shift2(st[0], k), _shift2(st[1], k)) + (c,) not in tset:
                raise ValueError("fold=True: the target Hamiltonian is not invariant under 2-site translations")


def _resolve_basis(k, sector, fold, basis) -> BasisSpec:
    N = 1 << (k - (1 if sector >= 0 else 0))
    if basis is not None:
        if fold:
            raise ValueError("pass either fold=True or an explicit basis, not both")
        if isinstance(basis, BasisSpec):
            return basis
        idx, w = basis if isinstance(basis, tuple) else (basis, None)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        if idx.size and (idx.min() < 0 or idx.max() >= N):
            raise ValueError("basis index out of range")
        return BasisSpec(int(idx.size), idx, None if w is None else np.ascontiguousarray(w, dtype=np.float64))
    if fold:
        return fold_basis(k, sector)
    return BasisSpec(N)


def _dist_info(distributed):
    if distributed is False:
        return 0, 1, None
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist.get_rank(), dist.get_world_size(), dist
    return 0, 1, None


def shard_chunks(nchunks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous chunk range of one rank (no data-path collective)."""
    lo = (nchunks * rank) // world
    hi = (nchunks * (rank + 1)) // world
    return lo, hi


def gather_records(local: torch.Tensor, lo: int, nchunks: int, rank: int, world: int, dist) -> torch.Tensor:
    """All-gather per-chunk records so every rank holds all chunks in order.

    Records are tiny (2 + 64 n_log doubles per chunk); the all-gather is the
    only collective of an evaluation (NCCL over NVLink, gloo in CPU tests)."""
    if dist is None:
        return local
    counts = [shard_chunks(nchunks, r, world) for r in range(world)]
    width = max(h - l for l, h in counts)
    # NCCL gathers device tensors; gloo (CPU tests, one-GPU boxes) gathers host copies
    dev = local.device if dist.get_backend() == "nccl" else torch.device("cpu")
    pad = torch.zeros((width, local.shape[1]), dtype=local.dtype, device=dev)
    pad[: local.shape[0]] = local.to(dev)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[: h - l] for b, (l, h) in zip(bufs, counts)], dim=0)


def ordered_sum(records: np.ndarray) -> np.ndarray:
    """Sum chunk records in ascending chunk order (deterministic)."""
    acc = np.zeros(records.shape[1], dtype=np.float64)
    for r in records:
        acc += r
    return acc


def _host_phi0(oracle, js_full: np.ndarray, k: int, sector: int) -> np.ndarray:
    """Generic duck-typed oracle (reference _phi_block, objective.py:561-565)."""
    rows = []
    sel = None
    if sector >= 0:
        i = np.arange(1 << (k - 1), dtype=np.int64)
        pc = np.array([bin(int(v)).count("1") & 1 for v in i], dtype=np.int64)
        sel = (i << 1) | (pc ^ sector)
    for j in js_full:
        col = np.conj(np.asarray(oracle.apply(basis_state(k, int(j))), dtype=np.complex128))
        rows.append(col if sel is None else col[sel])
    return np.ascontiguousarray(np.stack(rows))


class _Run:
    """One basis-sum evaluation (value / gradient / HVP) on this rank."""

    def __init__(self, circuit, oracle, flags, directions, sector, fold, basis, batch, chunk, distributed):
        self.k = circuit.num_qubits
        self.sector = _sector_code(sector)
        self.circuit = circuit
        self.flags = flags
        if fold:
            check_translation_invariant(circuit, oracle)
        self.spec = _resolve_basis(self.k, self.sector, fold, basis)
        self.N = 1 << (self.k - (1 if self.sector >= 0 else 0))
        total = self.spec.total
        self.batch = batch or _default_batch(self.N, max(total, 1))
        self.chunk = chunk or min(CHUNK_STATES, self.batch)
        if self.batch % self.chunk:
            self.batch = max(self.chunk, (self.batch // self.chunk) * self.chunk)
        self.rank, self.world, self.dist = _dist_info(distributed)
        self.plan = _get_plan(circuit, self.sector, self.batch, self.chunk)
        self.plan.set_gates(circuit.gate_stack())
        if flags & _lib.GF_HVP:
            self.plan.set_directions(directions)
        self.nd = self.plan.nd if flags & _lib.GF_HVP else 1
        self.rec = 2 + 32 * circuit.num_logical * (1 + self.nd)
        self.oracle = oracle

    def run(self):
        dev = self.plan.device
        total, chunk = self.spec.total, self.chunk
        nchunks = (total + chunk - 1) // chunk
        lo, hi = shard_chunks(nchunks, self.rank, self.world)
        rec = self.rec
        local = torch.zeros((hi - lo, rec), dtype=torch.float64, device=dev)
        phi0 = None  # allocated on the first batch the oracle has no resident rows for
        idx_all = None if self.spec.indices is None else torch.from_numpy(self.spec.indices).to(dev)
        w_all = None if self.spec.weights is None else torch.from_numpy(self.spec.weights).to(dev)
        launches = 0
        t0 = time.perf_counter()
        s0, s1 = lo * chunk, min(total, hi * chunk)
        pos = s0
        while pos < s1:
            nvec = min(self.batch, s1 - pos)
            if idx_all is None:
                basis = torch.arange(pos, pos + nvec, dtype=torch.int64, device=dev)
            else:
                basis = idx_all[pos:pos + nvec].contiguous()
            weights = None if w_all is None else w_all[pos:pos + nvec].contiguous()
            rows = getattr(self.oracle, "phi0_at", None)
            cur = rows(pos, nvec, self.sector, self.spec.indices) if rows is not None else None
            if cur is None:
                if phi0 is None:
                    phi0 = torch.empty((self.batch, self.N), dtype=torch.complex128, device=dev)
                self._fill_phi0(basis, phi0[:nvec])
                cur = phi0
            c0 = (pos // chunk) - lo
            nc = (nvec + chunk - 1) // chunk
            self.plan.eval(self.flags, nvec, basis, weights, cur, local[c0:c0 + nc])
            launches += self.plan.last_launches()
            pos += nvec
        # non-finite engine output -> FloatingPointError (GF_ENONFINITE)
        _lib.check(_lib.lib.gf_check_finite(local.data_ptr(), local.numel(), _lib.stream_ptr()))
        allrec = gather_records(local, lo, nchunks, self.rank, self.world, self.dist)
        host = allrec.cpu().numpy()
        self.elapsed = time.perf_counter() - t0
        self.launches = launches
        tot = ordered_sum(host) if host.shape[0] else np.zeros(rec)
        nlog = self.circuit.num_logical
        value = complex(tot[0], tot[1])
        d = tot[2:2 + 32 * nlog].view(np.complex128).reshape(nlog, 4, 4).copy()
        hs = tot[2 + 32 * nlog:].view(np.complex128).reshape(self.nd, nlog, 4, 4).copy()
        return value, d, (hs[0] if self.nd == 1 else hs)

    def _fill_phi0(self, basis: torch.Tensor, out: torch.Tensor):
        if self.sector >= 0:
            js_full = torch.empty_like(basis)
            _lib.check(_lib.lib.gf_sector_unrank(basis.data_ptr(), basis.numel(), self.sector, js_full.data_ptr(),
                                                 _lib.stream_ptr()))
        else:
            js_full = basis
        fn = getattr(self.oracle, "phi0_into", None)
        if fn is not None:
            fn(js_full, None if self.sector < 0 else self.sector, out)
            return
        host = _host_phi0(self.oracle, js_full.cpu().numpy(), self.k, self.sector)
        out.copy_(torch.from_numpy(host).to(out.device, non_blocking=False))


def _check_oracle(circuit, oracle):
    if oracle.num_qubits != circuit.num_qubits:
        raise ValueError(f"oracle acts on {oracle.num_qubits} qubits, circuit on {circuit.num_qubits}")


def _assert_bounded(value: float, bound: float):
    """Cauchy-Schwarz: f >= -(number of weighted summands) (reference
    objective.py:575-578 with Tr[I] = 2^k)."""
    if value < -bound * (1.0 + 1e-9) - 1e-9:
        raise FloatingPointError(f"objective {value} below the -{bound:g} trace bound")


def _riemannian(circuit, holo, parity_mode):
    euclid = [manifold.euclid_gradient_from_holomorphic(d) for d in holo]
    riem = [manifold.project_tangent_gate(g.matrix, e, parity_mode) for g, e in zip(circuit.logical_gates, euclid)]
    return euclid, riem


def _ref_counts(n: int, S: int, kind: str, pairs: int = 0, firsts: int = 0, arrays: int = 0):
    """Pass counters with the reference's semantics (objective.py:65-73)."""
    c = dict.fromkeys(COUNT_NAMES, 0)
    if kind == "value":
        c["gate_applications"] = n * S
    elif kind == "gradient":
        c["gate_applications"] = 2 * n * S
        c["hole_contractions"] = n * S
    elif kind == "hvp":
        c["gate_applications"] = (2 * n + 4 * max(n - 1, 0)) * S
        c["hole_contractions"] = 2 * max(n - 1, 0) * S
    elif kind == "hessian":
        c["gate_applications"] = 2 * n * S
        c["hole_contractions"] = n * S
        c["pair_contractions"] = pairs * S
        c["hole_applications"] = firsts * S
        c["array_gate_applications"] = arrays * S
    return c


def _slot_directions(circuit, directions):
    if len(directions) != circuit.num_logical:
        raise ValueError("need one direction matrix per logical gate")
    return np.ascontiguousarray(np.stack([np.asarray(z, dtype=np.complex128).reshape(4, 4) for z in directions]))


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------


def target_value(circuit: Circuit, oracle, workers: int | None = None, *, sector=None, fold=False, basis=None,
                 batch=None, chunk=None, distributed=None) -> float:
    """f = -Re Tr[U^dag C] (reference objective.py:586-608)."""
    _check_oracle(circuit, oracle)
    run = _Run(circuit, oracle, _lib.GF_VALUE, None, sector, fold, basis, batch, chunk, distributed)
    value, _, _ = run.run()
    f = float(-value.real)
    _assert_bounded(f, run.spec.weight_sum())
    return f


def _grad_report(circuit, run, value, holo, parity_mode, kind, t0, hvp=None):
    f = float(-value.real)
    _assert_bounded(f, run.spec.weight_sum())
    holo_l = [holo[i] for i in range(circuit.num_logical)]
    euclid, riem = _riemannian(circuit, holo_l, parity_mode)
    S = run.spec.total
    return ObjectiveReport(
        value=f,
        per_logical_gradient=riem,
        euclidean_gradients=euclid,
        holomorphic_derivatives=holo_l,
        wall_time=time.perf_counter() - t0,
        pass_counts=_ref_counts(circuit.num_slots, S, kind),
        engine={"launches": run.launches, "summands": S, "batch": run.batch, "chunk": run.chunk,
                "seconds": run.elapsed, "world": run.world, "weight_sum": run.spec.weight_sum()},
    )


def full_gradient(circuit: Circuit, oracle, workers: int | None = None, parity_mode: bool = False, *, sector=None,
                  fold=False, basis=None, batch=None, chunk=None, distributed=None) -> ObjectiveReport:
    """Value and Riemannian gradient per logical gate (reference
    objective.py:659-698)."""
    _check_oracle(circuit, oracle)
    t0 = time.perf_counter()
    run = _Run(circuit, oracle, _lib.GF_VALUE | _lib.GF_GRAD, None, sector, fold, basis, batch, chunk, distributed)
    value, d, _ = run.run()
    return _grad_report(circuit, run, value, d, parity_mode, "gradient", t0)


def gradient_and_hvp(circuit: Circuit, oracle, directions, parity_mode: bool = False, *, sector=None, fold=False,
                     basis=None, batch=None, chunk=None, distributed=None):
    """Fused value + gradient + one HVP in a single reversible 3-sweep pass
    (the bench's "gradient+HVP" evaluation).  Returns (report, hvp_list)."""
    _check_oracle(circuit, oracle)
    t0 = time.perf_counter()
    z = _slot_directions(circuit, directions)
    run = _Run(circuit, oracle, _lib.GF_VALUE | _lib.GF_GRAD | _lib.GF_HVP, z, sector, fold, basis, batch, chunk,
               distributed)
    value, d, h = run.run()
    rep = _grad_report(circuit, run, value, d, parity_mode, "gradient", t0)
    hv = _ref_counts(circuit.num_slots, run.spec.total, "hvp")
    rep.pass_counts = {k: rep.pass_counts[k] + hv[k] for k in COUNT_NAMES}
    return rep, [h[i] for i in range(circuit.num_logical)]


def _directions_per_sweep(circuit, sector) -> int:
    """HVP directions per set of sweeps (<= 3): each needs one more resident
    chi / v vector; at 2^31 amplitudes (32 GiB vectors) the device holds
    psi, bra, phi0 and at most two of them.  GF_DIRS_PER_SWEEP overrides."""
    env = os.environ.get("GF_DIRS_PER_SWEEP")
    if env:
        return int(max(1, min(3, int(env))))
    K = circuit.num_qubits - (1 if _sector_code(sector) >= 0 else 0)
    vec = 16 * (1 << K)
    if vec < (1 << 30):
        return 3
    if _sector_code(sector) >= 0 and os.environ.get("GF_SECTOR_FMA", "1") != "0":
        # parity sectors: single-direction sweeps run on the FMA unit engine, measured
        # faster than two directions per sweep on the DMMA path (c5: 70.2 s vs 78.7 s for 20 HVPs)
        return 1
    free, total = torch.cuda.mem_get_info()
    return int(max(1, min(3, total // vec - 3)))


def _multi_direction_ok(circuit, sector, batch, chunk, basis, fold) -> bool:
    """True when the plan for this evaluation runs the fused engine (the only
    one that evaluates several HVP directions per sweep)."""
    if os.environ.get("GF_ENGINE") == "stream":
        return False
    K = circuit.num_qubits - (1 if _sector_code(sector) >= 0 else 0)
    return K >= 6 and circuit.num_slots > 0


def hessian_vector_products(circuit: Circuit, oracle, direction_sets, *, sector=None, fold=False, basis=None,
                            batch=None, chunk=None, distributed=None):
    """Several HVPs with shared forward / reverse state sweeps: up to 3
    directions per set of sweeps on the fused engine (the full-Hessian
    columns).  Returns one list of per-logical 4x4 results per direction."""
    _check_oracle(circuit, oracle)
    zs = [_slot_directions(circuit, d) for d in direction_sets]
    out = []
    i = 0
    gmax = _directions_per_sweep(circuit, sector)
    while i < len(zs):
        group = zs[i:i + gmax]
        z = np.ascontiguousarray(np.stack(group)) if len(group) > 1 else group[0]
        if len(group) > 1 and not _multi_direction_ok(circuit, sector, batch, chunk, basis, fold):
            # the streaming engine (tiny state spaces, GF_ENGINE=stream) runs one direction per sweep
            group = group[:1]
            z = group[0]
        run = _Run(circuit, oracle, _lib.GF_HVP, z, sector, fold, basis, batch, chunk, distributed)
        _, _, h = run.run()
        hs = [h] if len(group) == 1 else list(h)
        out += [[x[j] for j in range(circuit.num_logical)] for x in hs]
        i += len(group)
    return out


def hessian_vector_product(circuit: Circuit, oracle, directions, workers: int | None = None, *, sector=None,
                           fold=False, basis=None, batch=None, chunk=None, distributed=None):
    """Holomorphic H~ . vec(Z) per logical gate (reference objective.py:770-814)."""
    _check_oracle(circuit, oracle)
    z = _slot_directions(circuit, directions)
    if not np.any(z) or circuit.num_slots == 0:
        return [np.zeros((4, 4), dtype=np.complex128) for _ in range(circuit.num_logical)]
    run = _Run(circuit, oracle, _lib.GF_HVP, z, sector, fold, basis, batch, chunk, distributed)
    _, _, h = run.run()
    return [h[i] for i in range(circuit.num_logical)]


def _pair_csr(circuit: Circuit, dedup: bool):
    """Slot pairs to contract, grouped by first slot, with multiplicity and
    logical-pair routing (reference objective.py:209-247): every ordered pair
    once, or one representative per translation class scaled by the class
    size when ``dedup`` (circuit.py:173-211)."""
    nlog = circuit.num_logical
    lids = [s.logical_id for s in circuit.slots]

    def route(a, b):
        return a * nlog - a * (a - 1) // 2 + (b - a)

    if dedup:
        pairs = translation_classes(circuit)
    else:
        n = circuit.num_slots
        pairs = [((a, b), 1) for a in range(n) for b in range(a + 1, n)]
    grouped: dict = {}
    for (a, b), mult in pairs:
        grouped.setdefault(a, []).append((b, mult))
    firsts = sorted(grouped)
    starts, seconds, mults, routes, syms, flips = [0], [], [], [], [], []
    for a in firsts:
        for b, mult in sorted(grouped[a]):
            la, lb = lids[a], lids[b]
            seconds.append(b)
            mults.append(float(mult))
            routes.append(route(min(la, lb), max(la, lb)))
            syms.append(la == lb)
            flips.append(la > lb)
        starts.append(len(seconds))
    return (np.array(firsts, np.int64), np.array(starts, np.int64), np.array(seconds, np.int64),
            np.array(mults, np.float64), np.array(routes, np.int64), np.array(syms, np.int32),
            np.array(flips, np.int32))


class HessianPlan:
    """Owns one gf_hess_plan: the reference's _hessian_chunk on the GPU
    (cached passes, hole arrays, pair contractions routed per the pair CSR)."""

    def __init__(self, circuit: Circuit, csr, support, batch: int, chunk: int):
        t1, t2, lid = circuit.slot_arrays()
        self.nlog = circuit.num_logical
        self.A = int(len(support))
        self.R = self.nlog * (self.nlog + 1) // 2
        self.rec = 2 + 32 * self.nlog + 2 * self.R * self.A * self.A
        self.batch, self.chunk = batch, chunk
        first, start, sec, mult, route, sym, flip = (np.ascontiguousarray(x) for x in csr)
        sup = np.ascontiguousarray(support, dtype=np.int64)
        self._keep = (t1, t2, lid, first, start, sec, mult, route, sym, flip, sup)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.gf_hess_plan_create(ctypes.byref(h), circuit.num_qubits, circuit.num_slots,
                                                t1.ctypes.data, t2.ctypes.data, lid.ctypes.data, self.nlog,
                                                sup.ctypes.data, self.A, first.ctypes.data, len(first),
                                                start.ctypes.data, sec.ctypes.data, mult.ctypes.data,
                                                route.ctypes.data, sym.ctypes.data, flip.ctypes.data, batch, chunk))
        self.h = h
        self.routes_used = sorted(set(int(r) for r in route))

    def set_gates(self, mats, parity_mode: bool):
        m = np.ascontiguousarray(mats, dtype=np.complex128)
        _lib.check(_lib.lib.gf_hess_plan_set_gates(self.h, m.ctypes.data, int(bool(parity_mode))))

    def eval(self, nvec, basis, weights, phi0, out, counts):
        _lib.check(_lib.lib.gf_hess_plan_eval(self.h, nvec, basis.data_ptr(),
                                              None if weights is None else weights.data_ptr(), phi0.data_ptr(),
                                              out.data_ptr(), counts.ctypes.data, _lib.stream_ptr()))

    def last_launches(self) -> int:
        return int(_lib.lib.gf_hess_plan_last_launches(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                _lib.lib.gf_hess_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass


class _RunInfo:
    """The fields _grad_report reads from a _Run."""

    def __init__(self, spec, info):
        self.spec = spec
        self.launches, self.batch, self.chunk = info["launches"], info["batch"], info["chunk"]
        self.elapsed, self.world = info["seconds"], info["world"]


def _full_hessian_pairs(circuit, oracle, dedup, parity_mode, basis, batch, chunk, distributed):
    """full_hessian through the pair-CSR chunk driver (reference
    objective.py:701-767): returns (value, holomorphic D per logical, blocks
    dict, counts, support, engine info)."""
    k = circuit.num_qubits
    spec = _resolve_basis(k, -1, False, basis)
    N = 1 << k
    n = circuit.num_slots
    sup = PARITY_SUPPORT if parity_mode else DENSE_SUPPORT
    A = len(sup)
    total = spec.total
    per = 16 * N * (2 * (n + 1) + 2 * A)  # cached passes + two hole arrays per summand
    if batch is None:
        env = os.environ.get("GF_BATCH")
        batch = int(env) if env else max(1, min(total, (8 << 30) // per))
    batch = max(1, min(batch, max(total, 1)))
    chunk = chunk or min(CHUNK_STATES, batch)
    if batch % chunk:
        batch = max(chunk, (batch // chunk) * chunk)
    csr = _pair_csr(circuit, dedup)
    hp = HessianPlan(circuit, csr, sup, batch, chunk)
    hp.set_gates(circuit.gate_stack(), parity_mode)
    rank, world, dist = _dist_info(distributed)
    dev = torch.device("cuda", torch.cuda.current_device())
    nchunks = (total + chunk - 1) // chunk
    lo, hi = shard_chunks(nchunks, rank, world)
    local = torch.zeros((hi - lo, hp.rec), dtype=torch.float64, device=dev)
    counts = np.zeros(5, np.int64)
    idx_all = None if spec.indices is None else torch.from_numpy(spec.indices).to(dev)
    w_all = None if spec.weights is None else torch.from_numpy(spec.weights).to(dev)
    phi0 = None
    launches = 0
    t0 = time.perf_counter()
    pos, s1 = lo * chunk, min(total, hi * chunk)
    while pos < s1:
        nvec = min(batch, s1 - pos)
        basis_t = (torch.arange(pos, pos + nvec, dtype=torch.int64, device=dev) if idx_all is None
                   else idx_all[pos:pos + nvec].contiguous())
        weights = None if w_all is None else w_all[pos:pos + nvec].contiguous()
        rows = getattr(oracle, "phi0_at", None)
        cur = rows(pos, nvec, -1, spec.indices) if rows is not None else None
        if cur is None:
            if phi0 is None:
                phi0 = torch.empty((batch, N), dtype=torch.complex128, device=dev)
            fn = getattr(oracle, "phi0_into", None)
            if fn is not None:
                fn(basis_t, None, phi0[:nvec])
            else:
                host = _host_phi0(oracle, basis_t.cpu().numpy(), k, -1)
                phi0[:nvec].copy_(torch.from_numpy(host).to(dev))
            cur = phi0
        c0 = (pos // chunk) - lo
        nc = (nvec + chunk - 1) // chunk
        hp.eval(nvec, basis_t, weights, cur, local[c0:c0 + nc], counts)
        launches += hp.last_launches()
        pos += nvec
    _lib.check(_lib.lib.gf_check_finite(local.data_ptr(), local.numel(), _lib.stream_ptr()))
    allrec = gather_records(local, lo, nchunks, rank, world, dist)
    host = allrec.cpu().numpy()
    tot = ordered_sum(host) if host.shape[0] else np.zeros(hp.rec)
    nlog = circuit.num_logical
    value = complex(tot[0], tot[1])
    d = tot[2:2 + 32 * nlog].view(np.complex128).reshape(nlog, 4, 4).copy()
    blk = tot[2 + 32 * nlog:].view(np.complex128).reshape(hp.R, A, A)
    blocks = {}
    for a in range(nlog):
        for b in range(a, nlog):
            r = a * nlog - a * (a - 1) // 2 + (b - a)
            if r in hp.routes_used:
                blocks[(a, b)] = blk[r].copy()
    if dist is not None:  # the counters of every rank's share
        ct = torch.from_numpy(counts).to(dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(ct)
        counts = ct.cpu().numpy()
    info = {"launches": launches, "summands": total, "batch": batch, "chunk": chunk,
            "seconds": time.perf_counter() - t0, "world": world, "weight_sum": spec.weight_sum(),
            "hessian_method": "pairs", "pairs": int(len(csr[2])), "dedup": bool(dedup)}
    return value, d, blocks, counts, sup, info


def _used_routes(circuit: Circuit):
    lid = [s.logical_id for s in circuit.slots]
    used = set()
    n = len(lid)
    for a in range(n):
        for b in range(a + 1, n):
            used.add((min(lid[a], lid[b]), max(lid[a], lid[b])))
    return used


def full_hessian(circuit: Circuit, oracle, use_translation_dedup: bool = False, parity_mode: bool = False,
                 workers: int | None = None, *, sector=None, fold=False, basis=None, batch=None, chunk=None,
                 distributed=None, method=None) -> ObjectiveReport:
    """Value, gradient and all holomorphic Hessian blocks (reference
    objective.py:701-767).

    Two engine algorithms (``method``):

    * ``"pairs"`` -- the reference's own: cached passes, a hole array per
      first slot propagated forward and contracted at every listed later slot
      (_hessian_chunk, objective.py:340-423) on the GPU
      (gf_hess_plan_eval).  With ``use_translation_dedup`` only one
      representative pair per translation class is contracted and scaled by
      the class size (the reference's work reduction).  Full space only.
    * ``"columns"`` -- blocks assembled column by column from engine HVPs with
      unit directions on the support entries (H~_{(a,i),(b,j)} =
      HVP(e_{b,j})[a][i]), three directions per set of reversible sweeps;
      supports ``sector`` / ``fold``.

    Default: "pairs" with ``use_translation_dedup`` (full space), else
    "columns" (measured faster without dedup, profiles/)."""
    _check_oracle(circuit, oracle)
    t0 = time.perf_counter()
    if method is None:
        method = "pairs" if (use_translation_dedup and sector is None and not fold) else "columns"
    if method not in ("pairs", "columns"):
        raise ValueError(f"unknown Hessian method {method!r}")
    if method == "pairs":
        if sector is not None or fold:
            raise ValueError("the pair-CSR Hessian runs in the full space (no sector / fold)")
        value, d, blocks, counts, sup, info = _full_hessian_pairs(circuit, oracle, use_translation_dedup,
                                                                  parity_mode, basis, batch, chunk, distributed)
        run = _RunInfo(_resolve_basis(circuit.num_qubits, -1, False, basis), info)
        rep = _grad_report(circuit, run, value, d, parity_mode, "gradient", t0)
        rep.engine.update(info)
        rep.hessian = HessianBlocks(circuit.num_logical, np.asarray(sup), blocks)
        rep.pass_counts = dict(zip(COUNT_NAMES, (int(c) for c in counts)))
        rep.wall_time = time.perf_counter() - t0
        return rep
    if use_translation_dedup:
        classes = translation_classes(circuit)
    rep = full_gradient(circuit, oracle, workers, parity_mode, sector=sector, fold=fold, basis=basis, batch=batch,
                        chunk=chunk, distributed=distributed)
    sup = PARITY_SUPPORT if parity_mode else DENSE_SUPPORT
    nlog = circuit.num_logical
    used = _used_routes(circuit)
    keys, dirs = [], []
    for b in range(nlog):
        if not any(b in key for key in used):
            continue
        for jj, e in enumerate(sup):
            z = np.zeros((nlog, 4, 4), dtype=np.complex128)
            z[b].reshape(16)[e] = 1.0
            keys.append((b, jj))
            dirs.append(z)
    # columns in sweeps of up to 3 unit directions sharing the psi / bra work
    res = hessian_vector_products(circuit, oracle, dirs, sector=sector, fold=fold, basis=basis, batch=batch,
                                  chunk=chunk, distributed=distributed)
    cols = dict(zip(keys, res))
    blocks = {}
    for a, b in sorted(used):
        blk = np.empty((sup.size, sup.size), dtype=np.complex128)
        for jj in range(sup.size):
            blk[:, jj] = cols[(b, jj)][a].reshape(16)[sup]
        blocks[(a, b)] = blk
    rep.hessian = HessianBlocks(nlog, np.asarray(sup), blocks)
    n = circuit.num_slots
    pairs = len(classes) if use_translation_dedup else n * (n - 1) // 2
    S = rep.engine.get("summands", 0)
    rep.pass_counts = _ref_counts(n, S, "hessian", pairs=pairs, firsts=max(n - 1, 0),
                                  arrays=max(n - 1, 0) * max(n - 2, 0) // 2)
    rep.wall_time = time.perf_counter() - t0
    return rep


def build_pass_cache(circuit: Circuit, oracle, j: int) -> PassCache:
    """Forward / backward states of summand j (reference objective.py:611-624),
    computed with the GPU gate kernel."""
    _check_oracle(circuit, oracle)
    k = circuit.num_qubits
    fwd = [basis_state(k, j)]
    for s in circuit.slots:
        fwd.append(apply_gate(fwd[-1], Gate(circuit.logical_gates[s.logical_id].matrix, s.targets)))
    bwd = [np.conj(oracle.apply(basis_state(k, j)))]
    for s in reversed(circuit.slots):
        bwd.append(apply_gate(bwd[-1], Gate(circuit.logical_gates[s.logical_id].matrix.T, s.targets)))
    return PassCache(fwd, bwd)


def summand_gradient(j: int, circuit: Circuit, oracle):
    """(value, per-slot holomorphic derivatives) of summand j (reference
    objective.py:627-642)."""
    if not 0 <= j < 2**circuit.num_qubits:
        raise ValueError(f"basis index {j} out of range")
    cache = build_pass_cache(circuit, oracle, j)
    n = circuit.num_slots
    value = complex(cache.backward_states[0] @ cache.forward_states[-1])
    derivs = [hole_contract(cache.backward_states[n - l - 1], cache.forward_states[l], s.targets)
              for l, s in enumerate(circuit.slots)]
    return value, derivs


def _unswap(d, swapped):
    return d[np.ix_(WIRE_SWAP, WIRE_SWAP)] if swapped else d


__all__ += ["accumulate_shared"]
