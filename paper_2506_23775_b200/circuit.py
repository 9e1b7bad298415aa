"""Circuit topology: ordered slots sharing logical gates (host-side data model).

Same semantics as the reference ``gatefit.circuit`` (reference circuit.py:30-211):
slots apply in list order to the input state; several slots may share one
logical gate and their derivatives are summed onto it.  Checkpoint file IO
(reference circuit.py:219-312) is a file format, not engine compute, and is
out of scope for this drop-in.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kernels import Gate

__all__ = [
    "GateSlot",
    "BrickwallMeta",
    "Circuit",
    "build_brickwall",
    "circuit_apply",
    "accumulate_shared",
    "translation_classes",
    "brickwall_bonds",
]


@dataclass(frozen=True)
class GateSlot:
    logical_id: int
    targets: tuple[int, int]


@dataclass(frozen=True)
class BrickwallMeta:
    num_layers: int
    layer_of_slot: tuple[int, ...]
    translation_period: int = 2
    periodic: bool = False


@dataclass
class Circuit:
    """Slot list + logical gates (reference circuit.py:48-88)."""

    num_qubits: int
    slots: list[GateSlot]
    logical_gates: list[Gate]
    topology: BrickwallMeta | None = None

    def __post_init__(self):
        nlog = len(self.logical_gates)
        k = self.num_qubits
        for s in self.slots:
            if s.logical_id < 0 or s.logical_id >= nlog:
                raise ValueError(f"slot references unknown logical gate {s.logical_id}")
            a, b = s.targets
            if a == b or min(a, b) < 0 or max(a, b) >= k:
                raise ValueError(f"invalid slot targets {s.targets}")

    @property
    def num_slots(self) -> int:
        return len(self.slots)

    @property
    def num_logical(self) -> int:
        return len(self.logical_gates)

    def slot_matrix(self, index: int) -> np.ndarray:
        return self.logical_gates[self.slots[index].logical_id].matrix

    def with_gates(self, matrices) -> "Circuit":
        if len(matrices) != self.num_logical:
            raise ValueError("need one matrix per logical gate")
        new = [Gate(m, g.targets, g.parity_sparse) for g, m in zip(self.logical_gates, matrices)]
        return Circuit(self.num_qubits, self.slots, new, self.topology)

    # flat views consumed by the engine plan
    def slot_arrays(self):
        t = np.array([s.targets for s in self.slots], dtype=np.int32).reshape(-1, 2)
        lid = np.array([s.logical_id for s in self.slots], dtype=np.int32)
        return np.ascontiguousarray(t[:, 0]), np.ascontiguousarray(t[:, 1]), lid

    def gate_stack(self) -> np.ndarray:
        if not self.logical_gates:
            return np.zeros((0, 4, 4), np.complex128)
        return np.ascontiguousarray(np.stack([g.matrix for g in self.logical_gates]), dtype=np.complex128)


def brickwall_bonds(num_qubits: int, layer: int, periodic: bool) -> list[tuple[int, int]]:
    """Even layers: (0,1),(2,3),...; odd layers: (1,2),(3,4),... plus the wrap
    bond (L-1, 0) when periodic (reference circuit.py:121-127)."""
    if layer % 2 == 0:
        return [(j, j + 1) for j in range(0, num_qubits, 2)]
    out = [(j, j + 1) for j in range(1, num_qubits - 1, 2)]
    if periodic:
        out.append((num_qubits - 1, 0))
    return out


def build_brickwall(num_qubits: int, num_layers: int, initial_gates, periodic: bool = False) -> Circuit:
    """One shared logical gate per layer (reference circuit.py:91-118)."""
    if num_qubits < 2 or num_qubits % 2:
        raise ValueError("brick wall requires an even number of qubits >= 2")
    if len(initial_gates) != num_layers:
        raise ValueError("need exactly one initial gate per layer")
    gates = [g if isinstance(g, Gate) else Gate(g, (0, 1)) for g in initial_gates]
    slots, layer_of = [], []
    for layer in range(num_layers):
        for bond in brickwall_bonds(num_qubits, layer, periodic):
            slots.append(GateSlot(layer, bond))
            layer_of.append(layer)
    return Circuit(num_qubits, slots, gates, BrickwallMeta(num_layers, tuple(layer_of), 2, periodic))


def circuit_apply(circuit: Circuit, state, direction: str = "forward"):
    """Apply the circuit (or its reversed transposed form) on the GPU."""
    import torch

    from .kernels import _finish, _lib, _stage

    if direction not in ("forward", "backward_transposed"):
        raise ValueError(f"unknown direction {direction!r}")
    s, host = _stage(state, 1)
    if s.shape[0] != 1 << circuit.num_qubits:
        raise ValueError("state dimension does not match circuit qubit count")
    cur = s.clone()
    order = range(circuit.num_slots)
    if direction == "backward_transposed":
        order = reversed(order)
    for i in order:
        slot = circuit.slots[i]
        m = circuit.logical_gates[slot.logical_id].matrix
        if direction == "backward_transposed":
            m = m.T
        m = np.ascontiguousarray(m, dtype=np.complex128)
        _lib.check(_lib.lib.gf_apply_gate(cur.data_ptr(), cur.data_ptr(), circuit.num_qubits, slot.targets[0],
                                          slot.targets[1], m.ctypes.data, 0, 1, _lib.stream_ptr()))
    torch.cuda.current_stream().synchronize()
    return _finish(cur, host)


def accumulate_shared(per_slot_grads, circuit: Circuit):
    """Sum per-slot matrices onto logical gates (reference circuit.py:161-170)."""
    if len(per_slot_grads) != circuit.num_slots:
        raise ValueError("need exactly one gradient matrix per slot")
    acc = np.zeros((circuit.num_logical, 4, 4), dtype=np.complex128)
    for slot, g in zip(circuit.slots, per_slot_grads):
        acc[slot.logical_id] += g
    return list(acc)


def translation_classes(circuit: Circuit, policy: str = "lex_min"):
    """Orbits of ordered slot pairs under translations by multiples of the
    brick-wall period (reference circuit.py:173-211): list of
    ``((a, b), class_size)`` sorted by representative."""
    meta = circuit.topology
    if meta is None or not meta.periodic:
        raise ValueError("translation classes require a periodic brick-wall circuit")
    if policy not in ("lex_min", "lex_max"):
        raise ValueError(f"unknown representative policy {policy!r}")
    L = circuit.num_qubits
    where = {(meta.layer_of_slot[i], s.targets[0]): i for i, s in enumerate(circuit.slots)}
    shifts = list(range(0, L, meta.translation_period))
    n = circuit.num_slots
    # image of each slot under each shift
    img = np.array([[where[(meta.layer_of_slot[i], (circuit.slots[i].targets[0] + d) % L)] for d in shifts]
                    for i in range(n)], dtype=np.int64).reshape(n, len(shifts))
    choose = min if policy == "lex_min" else max
    counts: dict[tuple[int, int], int] = {}
    for a in range(n):
        for b in range(a + 1, n):
            ia, ib = img[a], img[b]
            orbit = [(int(x), int(y)) if x < y else (int(y), int(x)) for x, y in zip(ia, ib)]
            rep = choose(orbit)
            counts[rep] = counts.get(rep, 0) + 1
    return sorted(counts.items())
