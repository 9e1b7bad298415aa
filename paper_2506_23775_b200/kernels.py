"""Public contraction primitives, executed by the sm_100a kernels of libgfcuda.so.

Mirrors the public surface of the reference ``gatefit.kernels``
(reference kernels.py:25-47 and kernels.py:484-623): same names, argument
meaning, orientation conventions and ``ValueError`` cases.  Host ``numpy``
inputs are staged through device memory and returned as ``numpy``; CUDA
``torch`` tensors stay on the device (zero copy) and are returned as tensors.

Conventions (reference kernels.py:1-22): qubit 0 is the most significant bit,
gate index ``2*b(t1) + b(t2)``, hole arrays ``[2**k, arity]`` with the arity
index fastest.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "Gate",
    "WIRE_SWAP",
    "DENSE_SUPPORT",
    "PARITY_SUPPORT",
    "support_table",
    "num_qubits",
    "basis_state",
    "leg_dims",
    "wire_swapped_matrix",
    "apply_gate",
    "hole_contract",
    "hole_apply",
    "apply_gate_to_array",
    "hole_contract_array",
    "apply_sector_c1q",
    "apply_gate_1q",
]

#: wire exchange permutation of a 4x4 gate's rows / columns (kernels.py:49-50)
WIRE_SWAP = np.array([0, 2, 1, 3], dtype=np.int64)
#: flat entries 4*row+col kept by a dense / parity-conserving hole (kernels.py:52-58)
DENSE_SUPPORT = np.arange(16, dtype=np.int64)
PARITY_SUPPORT = np.array([0, 3, 5, 6, 9, 10, 12, 15], dtype=np.int64)
_OFF_PATTERN = np.array([1, 2, 4, 7, 8, 11, 13, 14])


@dataclass
class Gate:
    """4x4 gate matrix on an ordered qubit pair (reference kernels.py:61-80)."""

    matrix: np.ndarray
    targets: tuple[int, int]
    parity_sparse: bool = False

    def __post_init__(self):
        m = np.ascontiguousarray(self.matrix, dtype=np.complex128)
        if m.shape != (4, 4):
            raise ValueError(f"gate matrix must be 4x4, got {m.shape}")
        a, b = (int(x) for x in self.targets)
        if a == b:
            raise ValueError("gate targets must be distinct qubits")
        self.matrix = m
        self.targets = (a, b)


def num_qubits(state) -> int:
    n = int(state.shape[0])
    k = n.bit_length() - 1
    if n <= 0 or (1 << k) != n:
        raise ValueError(f"state length {n} is not a power of two")
    return k


def basis_state(k: int, j: int) -> np.ndarray:
    if not 0 <= j < (1 << k):
        raise ValueError(f"basis index {j} out of range for {k} qubits")
    v = np.zeros(1 << k, dtype=np.complex128)
    v[j] = 1.0
    return v


def leg_dims(k: int, q1: int, q2: int) -> tuple[int, int, int]:
    """(p, q, n) environment legs of a gate on q1 < q2 (kernels.py:99-101)."""
    return 1 << q1, 1 << (q2 - q1 - 1), 1 << (k - 1 - q2)


def wire_swapped_matrix(matrix: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(matrix)[np.ix_(WIRE_SWAP, WIRE_SWAP)])


def support_table(support) -> tuple[np.ndarray, np.ndarray]:
    s = np.asarray(support, dtype=np.int64)
    return s // 4, s % 4


def _is_parity(m: np.ndarray) -> bool:
    return bool(np.all(m.reshape(16)[_OFF_PATTERN] == 0))


# ---------------------------------------------------------------- staging


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_23775_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stage(x, ndim):
    """-> (contiguous complex128 CUDA tensor, came_from_numpy)."""
    if isinstance(x, torch.Tensor):
        if x.ndim != ndim:
            raise ValueError(f"expected a {ndim}-D array, got shape {tuple(x.shape)}")
        t = x
        if not t.is_cuda:
            t = t.to(_device())
        return t.to(torch.complex128).contiguous(), False
    a = np.asarray(x)
    if a.ndim != ndim:
        raise ValueError(f"expected a {ndim}-D array, got shape {a.shape}")
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return torch.from_numpy(a).to(_device()), True


def _finish(t, to_numpy):
    if to_numpy:
        return t.cpu().numpy()
    return t


def _mat_ptr(m):
    m = np.ascontiguousarray(m, dtype=np.complex128)
    return m, m.ctypes.data


# ---------------------------------------------------------------- ops


def apply_gate(state, gate: Gate, out=None, variant: str = "kernel"):
    """``out = G state`` (reference kernels.py:484-515).

    ``variant`` is accepted for API parity; "kernel" and "plain" are the same
    GPU kernel (bit-identical, as the reference requires of its two loop
    orders)."""
    if variant not in ("kernel", "plain"):
        raise ValueError(f"unknown kernel variant {variant!r}")
    s, host = _stage(state, 1)
    k = num_qubits(s)
    if out is not None:
        if out is state or (isinstance(out, np.ndarray) and isinstance(state, np.ndarray)
                            and np.may_share_memory(out, state)):
            raise ValueError("output buffer must not alias the input state")
        if isinstance(out, torch.Tensor) and isinstance(state, torch.Tensor) and out.data_ptr() == state.data_ptr():
            raise ValueError("output buffer must not alias the input state")
    res = torch.empty_like(s)
    m, mp = _mat_ptr(gate.matrix)
    _lib.check(_lib.lib.gf_apply_gate(s.data_ptr(), res.data_ptr(), k, gate.targets[0], gate.targets[1], mp,
                                      int(_is_parity(m)), 1, _lib.stream_ptr()))
    if out is not None:
        if isinstance(out, torch.Tensor):
            out.copy_(res)
        else:
            out[...] = res.cpu().numpy()
        return out
    return _finish(res, host)


def apply_gate_1q(state, matrix, qubit: int):
    """``g state`` for a 2x2 gate on one qubit (north-star item 1; the
    reference embeds 1q gates in its 2q gates)."""
    s, host = _stage(state, 1)
    k = num_qubits(s)
    g = np.ascontiguousarray(matrix, dtype=np.complex128)
    if g.shape != (2, 2):
        raise ValueError(f"one-qubit gate must be 2x2, got {g.shape}")
    res = torch.empty_like(s)
    _lib.check(_lib.lib.gf_apply_gate_1q(s.data_ptr(), res.data_ptr(), k, int(qubit), g.ctypes.data, 1,
                                         _lib.stream_ptr()))
    return _finish(res, host)


def apply_sector_c1q(state, matrix, a: int, k_full: int, sector: int = 0):
    """Parity-controlled one-qubit gate on a sector-compressed vector: the
    4x4 parity-conserving ``matrix`` on full-space qubits (a, k_full-1)."""
    s, host = _stage(state, 1)
    if s.shape[0] != 1 << (k_full - 1):
        raise ValueError("compressed state must have 2**(k_full-1) amplitudes")
    res = torch.empty_like(s)
    m, mp = _mat_ptr(matrix)
    _lib.check(_lib.lib.gf_apply_gate_sector_c1q(s.data_ptr(), res.data_ptr(), k_full, a, sector, mp, 1,
                                                 _lib.stream_ptr()))
    return _finish(res, host)


def hole_contract(bra, ket, targets):
    """Environment D with ``sum(G * D) == bra . (G ket)`` (kernels.py:518-537)."""
    b, host = _stage(bra, 1)
    kt, _ = _stage(ket, 1)
    if b.shape != kt.shape:
        raise ValueError("bra and ket must have the same length")
    k = num_qubits(b)
    out = torch.empty(16, dtype=torch.complex128, device=b.device)
    _lib.check(_lib.lib.gf_hole_contract(b.data_ptr(), kt.data_ptr(), k, int(targets[0]), int(targets[1]), 1,
                                         out.data_ptr(), _lib.stream_ptr()))
    return _finish(out.reshape(4, 4), host)


def hole_apply(state, targets, support=None):
    """Hole array ``[2**k, arity]`` (kernels.py:540-565)."""
    s, host = _stage(state, 1)
    k = num_qubits(s)
    sup = np.ascontiguousarray(DENSE_SUPPORT if support is None else support, dtype=np.int64)
    out = torch.empty((s.shape[0], sup.size), dtype=torch.complex128, device=s.device)
    _lib.check(_lib.lib.gf_hole_apply(s.data_ptr(), out.data_ptr(), k, int(targets[0]), int(targets[1]),
                                      sup.ctypes.data, int(sup.size), _lib.stream_ptr()))
    return _finish(out, host)


def apply_gate_to_array(array, gate: Gate, out=None):
    """Gate on every logical vector of a hole array (kernels.py:574-597)."""
    arr, host = _stage(array, 2)
    k = num_qubits(arr)
    if out is not None and (out is array or (isinstance(out, np.ndarray) and isinstance(array, np.ndarray)
                                              and np.may_share_memory(out, array))):
        raise ValueError("output buffer must not alias the input array")
    res = torch.empty_like(arr)
    m, mp = _mat_ptr(gate.matrix)
    _lib.check(_lib.lib.gf_apply_gate_to_array(arr.data_ptr(), res.data_ptr(), k, int(arr.shape[1]),
                                               gate.targets[0], gate.targets[1], mp, int(_is_parity(m)),
                                               _lib.stream_ptr()))
    if out is not None:
        if isinstance(out, torch.Tensor):
            out.copy_(res)
        else:
            out[...] = res.cpu().numpy()
        return out
    return _finish(res, host)


def hole_contract_array(bra, ket_array, targets, support=None):
    """``B[a, c] = hole_contract(bra, ket_array[:, a]).flat[support[c]]``
    (kernels.py:600-623)."""
    b, host = _stage(bra, 1)
    arr, _ = _stage(ket_array, 2)
    if arr.shape[0] != b.shape[0]:
        raise ValueError("ket array must have shape (len(bra), arity)")
    k = num_qubits(b)
    sup = np.ascontiguousarray(DENSE_SUPPORT if support is None else support, dtype=np.int64)
    A = int(arr.shape[1])
    out = torch.empty((A, sup.size), dtype=torch.complex128, device=b.device)
    _lib.check(_lib.lib.gf_hole_contract_array(b.data_ptr(), arr.data_ptr(), k, A, int(targets[0]),
                                               int(targets[1]), sup.ctypes.data, int(sup.size), out.data_ptr(),
                                               _lib.stream_ptr()))
    return _finish(out, host)
