"""CPU tests of the fused-pass planner (host code in libgfcuda.so, queried
through gf_plan_layout without any device work).

A fused pass runs several slots on one shared-memory tile. The planner must
keep every ordering the sweep needs: any two slots that share a qubit (or,
in a parity sector, that both act on the implicit qubit) run in sweep order,
as in the reference's slot loop (objective.py:255-280, 291-337). Each pass's
slots must fit its m local bits, which always include the c = 3 lowest
physical bits (contiguous 128 B runs)."""

import ctypes
import os

import numpy as np
import pytest

from paper_2506_23775_b200 import _lib
from paper_2506_23775_b200 import models

MAXP = 256


def layout(circ, sector, m, sweep, env=None):
    t1, t2, _ = circ.slot_arrays()
    k = circ.num_qubits
    np_ = ctypes.c_int(0)
    sizes = np.zeros(MAXP, np.int32)
    order = np.zeros(circ.num_slots, np.int32)
    bits = np.zeros(MAXP, np.uint64)
    old = {}
    for kk, v in (env or {}).items():
        old[kk] = os.environ.get(kk)
        os.environ[kk] = v
    try:
        _lib.check(_lib.lib.gf_plan_layout(k, sector, circ.num_slots, t1.ctypes.data, t2.ctypes.data, m, sweep, MAXP,
                                           ctypes.byref(np_), sizes.ctypes.data, order.ctypes.data, bits.ctypes.data))
    finally:
        for kk, v in old.items():
            if v is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = v
    n = np_.value
    return sizes[:n].tolist(), order.tolist(), [int(b) for b in bits[:n]]


def slot_bits(circ, sector, s):
    """Physical bit positions a slot touches, plus a virtual bit 63 for gates
    on a parity sector's implicit qubit (those never reorder)."""
    t1, t2, _ = circ.slot_arrays()
    k = circ.num_qubits
    K = k - 1 if sector >= 0 else k
    a, b = sorted((int(t1[s]), int(t2[s])))
    if sector >= 0 and b == k - 1:
        return {K - 1 - a}, {K - 1 - a, 63}
    bs = {K - 1 - b, K - 1 - a}
    return bs, bs


def check_plan_env(circ, sector, m, sweep, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return check_plan(circ, sector, m, sweep)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def check_plan(circ, sector, m, sweep):
    sizes, order, pbits = layout(circ, sector, m, sweep)
    n = circ.num_slots
    assert sum(sizes) == n and sorted(order) == list(range(n))   # every slot exactly once
    assert all(1 <= s <= 16 for s in sizes)
    pos = {s: i for i, s in enumerate(order)}
    seq = list(range(n)) if sweep == 0 else list(range(n - 1, -1, -1))
    # dependency order: slots sharing a (virtual) qubit keep sweep order
    for i in range(n):
        for j in range(i + 1, n):
            a, b = seq[i], seq[j]
            if slot_bits(circ, sector, a)[1] & slot_bits(circ, sector, b)[1]:
                assert pos[a] < pos[b], (a, b)
    # each pass: m local bits including the 3 lowest, covering its slots' bits
    o = 0
    for sz, bits in zip(sizes, pbits):
        assert bin(bits).count("1") == min(m, circ.num_qubits - (1 if sector >= 0 else 0))
        assert bits & 0b111 == 0b111
        for s in order[o:o + sz]:
            assert all((bits >> q) & 1 for q in slot_bits(circ, sector, s)[0])
        o += sz
    return sizes


@pytest.mark.parametrize("sweep", [0, 1])
def test_c2_plan_is_three_passes_and_valid(sweep):
    # BASELINE configs[1]: L=8 spinful, 5 layers, 16 qubits, 36 slots; the exact
    # beam over local sets finds 3 passes per sweep (the greedy search needs 4)
    _, circ, _ = models.spinful_layer_circuit(8, 5, False, seed=1)
    sizes = check_plan_env(circ, -1, 11, sweep, {"GF_PLAN_MINPASS": "1"})
    assert len(sizes) == 3
    greedy, _, _ = layout(circ, -1, 11, sweep, env={"GF_PLAN_GREEDY": "1"})
    assert len(greedy) >= len(sizes)
    # default: with the light-cone rule dead tiles are free, so the planner may
    # spend one more pass near the |j> end when that leaves less live slot work
    lc = check_plan(circ, -1, 11, sweep)
    assert len(sizes) <= len(lc) <= len(sizes) + 1 and sum(lc) == sum(sizes) == 36


@pytest.mark.parametrize("L,layers,periodic,sector,m", [
    (4, 3, False, -1, 5), (6, 4, True, 0, 6), (6, 5, False, 1, 7), (12, 7, False, 0, 11), (8, 5, False, -1, 8),
])
def test_plans_respect_slot_order_and_local_bits(L, layers, periodic, sector, m):
    _, circ, _ = models.spinful_layer_circuit(L, layers, periodic, seed=0, parity=sector >= 0)
    for sweep in (0, 1):
        check_plan(circ, sector, m, sweep)


def test_layout_rejects_bad_queries():
    _, circ, _ = models.spinful_layer_circuit(4, 2, False, seed=0)
    t1, t2, _ = circ.slot_arrays()
    bad = np.array(t2, np.int32)
    bad[0] = t1[0]
    z = np.zeros(64, np.int32)
    b = np.zeros(64, np.uint64)
    n = ctypes.c_int(0)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib.gf_plan_layout(circ.num_qubits, -1, circ.num_slots, t1.ctypes.data, bad.ctypes.data, 6, 0,
                                           64, ctypes.byref(n), z.ctypes.data, z.ctypes.data, b.ctypes.data))
    with pytest.raises(ValueError):  # no room for the passes
        _lib.check(_lib.lib.gf_plan_layout(circ.num_qubits, -1, circ.num_slots, t1.ctypes.data, t2.ctypes.data, 5, 0,
                                           0, ctypes.byref(n), z.ctypes.data, z.ctypes.data, b.ctypes.data))
