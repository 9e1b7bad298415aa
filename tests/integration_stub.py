"""The reference-side ctypes stub of INTEGRATION.md section B, verbatim except
for the library path.  tests/test_gpu_engine.py::test_integration_stub drives it
exactly as the reference's objective.py chunk closure would."""
# gatefit/_b200.py -- route the per-chunk drivers to libgfcuda.so
import ctypes
import numpy as np

import os
_lib = ctypes.CDLL(os.environ.get("GF_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_23775_b200", "libgfcuda.so")))
_vp, _i, _i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
_lib.gf_last_error.restype = ctypes.c_char_p
for name, args in {
    "gf_plan_create": [ctypes.POINTER(_vp), _i, _i, _i, _vp, _vp, _vp, _i, _i64, _i],
    "gf_plan_set_gates": [_vp, _vp], "gf_plan_set_directions": [_vp, _vp],
    "gf_plan_eval": [_vp, _i, _i64, _vp, _vp, _vp, _vp, _vp],
    "gf_plan_slot_outputs": [_vp, _i64, _vp, _vp, _vp], "gf_plan_destroy": [_vp],
    "gf_malloc": [ctypes.POINTER(_vp), _i64], "gf_free": [_vp],
    "gf_memcpy": [_vp, _vp, _i64, _i, _vp], "gf_stream_sync": [_vp],
}.items():
    getattr(_lib, name).argtypes = args
    getattr(_lib, name).restype = _i
GF_VALUE, GF_GRAD, GF_HVP = 1, 2, 4
H2D, D2H = 0, 1


def _check(rc):
    if rc:
        msg = _lib.gf_last_error().decode()
        raise {1: ValueError, 2: FloatingPointError, 4: MemoryError}.get(rc, RuntimeError)(msg)


def _dev(nbytes):
    p = _vp()
    _check(_lib.gf_malloc(ctypes.byref(p), nbytes))
    return p


class GpuChunkEvaluator:
    """One plan per circuit topology; evaluates [j0, j1) like the numba drivers."""

    def __init__(self, circuit, max_chunk=64):
        k, n = circuit.num_qubits, circuit.num_slots
        t1 = np.array([s.targets[0] for s in circuit.slots], np.int32)
        t2 = np.array([s.targets[1] for s in circuit.slots], np.int32)
        lid = np.array([s.logical_id for s in circuit.slots], np.int32)
        self.k, self.n, self.N, self.max = k, n, 1 << k, max_chunk
        self.h = _vp()
        _check(_lib.gf_plan_create(ctypes.byref(self.h), k, -1, n, t1.ctypes.data, t2.ctypes.data,
                                   lid.ctypes.data, circuit.num_logical, max_chunk, max_chunk))
        mats = np.ascontiguousarray(np.stack([g.matrix for g in circuit.logical_gates]), np.complex128)
        _check(_lib.gf_plan_set_gates(self.h, mats.ctypes.data))
        self.basis = _dev(8 * max_chunk)
        self.phi0 = _dev(16 * self.N * max_chunk)
        self.rec = _dev(8 * (2 + 64 * circuit.num_logical))
        self.slots = _dev(2 * 16 * 16 * n)

    def set_directions(self, zmats):             # [n_logical, 4, 4], logical orientation
        z = np.ascontiguousarray(zmats, np.complex128)
        _check(_lib.gf_plan_set_directions(self.h, z.ctypes.data))

    def __call__(self, flags, j0, j1, phi0s):
        """Returns (value, dacc[n,4,4], oacc[n,4,4]) with the semantics of
        _gradient_chunk / _hvp_chunk (objective.py:322-337, 432-482)."""
        J = j1 - j0
        js = np.arange(j0, j1, dtype=np.int64)
        phi = np.ascontiguousarray(phi0s, np.complex128)
        _check(_lib.gf_memcpy(self.basis, js.ctypes.data, js.nbytes, H2D, None))
        _check(_lib.gf_memcpy(self.phi0, phi.ctypes.data, phi.nbytes, H2D, None))
        _check(_lib.gf_plan_eval(self.h, flags, J, self.basis, None, self.phi0, self.rec, None))
        _check(_lib.gf_plan_slot_outputs(self.h, J, self.slots, ctypes.c_void_p(self.slots.value + 16 * 16 * self.n), None))
        val = np.empty(2)
        sl = np.empty((2, self.n, 4, 4), np.complex128)
        _check(_lib.gf_memcpy(val.ctypes.data, self.rec, 16, D2H, None))
        _check(_lib.gf_memcpy(sl.ctypes.data, self.slots, sl.nbytes, D2H, None))
        _check(_lib.gf_stream_sync(None))
        return complex(val[0], val[1]), sl[0], sl[1]


for name, args in {
    "gf_hess_plan_create": [ctypes.POINTER(_vp), _i, _i, _vp, _vp, _vp, _i, _vp, _i, _vp, _i64, _vp, _vp, _vp, _vp,
                            _vp, _vp, _i64, _i],
    "gf_hess_plan_set_gates": [_vp, _vp, _i],
    "gf_hess_plan_eval": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "gf_hess_plan_slot_outputs": [_vp, _i64, _vp, _vp], "gf_hess_plan_destroy": [_vp],
}.items():
    getattr(_lib, name).argtypes = args
    getattr(_lib, name).restype = _i


class GpuHessianChunkEvaluator:
    """_hessian_chunk (objective.py:340-423) on the GPU: built from the
    reference's own _Plan support and _pair_csr output."""

    def __init__(self, circuit, support, csr, parity_mode=False, max_chunk=64):
        k, n, nlog = circuit.num_qubits, circuit.num_slots, circuit.num_logical
        t1 = np.array([s.targets[0] for s in circuit.slots], np.int32)
        t2 = np.array([s.targets[1] for s in circuit.slots], np.int32)
        lid = np.array([s.logical_id for s in circuit.slots], np.int32)
        first, start, sec, mult, route, sym, flip = csr
        keep = [np.ascontiguousarray(x, dt) for x, dt in ((first, np.int64), (start, np.int64), (sec, np.int64),
                                                           (mult, np.float64), (route, np.int64), (sym, np.int32),
                                                           (flip, np.int32))]
        sup = np.ascontiguousarray(support, np.int64)
        self.n, self.N, self.A = n, 1 << k, len(sup)
        self.R = nlog * (nlog + 1) // 2
        self.rec = 2 + 32 * nlog + 2 * self.R * self.A * self.A
        self.h = _vp()
        _check(_lib.gf_hess_plan_create(ctypes.byref(self.h), k, n, t1.ctypes.data, t2.ctypes.data, lid.ctypes.data,
                                        nlog, sup.ctypes.data, self.A, keep[0].ctypes.data, len(keep[0]),
                                        *[x.ctypes.data for x in keep[1:]], max_chunk, max_chunk))
        mats = np.ascontiguousarray(np.stack([g.matrix for g in circuit.logical_gates]), np.complex128)
        _check(_lib.gf_hess_plan_set_gates(self.h, mats.ctypes.data, int(parity_mode)))
        self.basis = _dev(8 * max_chunk)
        self.phi0 = _dev(16 * self.N * max_chunk)
        self.out = _dev(8 * self.rec)
        self.slots = _dev(16 * 16 * n)

    def __call__(self, j0, j1, phi0s):
        """Returns (value, dacc[n,4,4], block_acc[R,A,A], counts[5]) like
        _hessian_chunk plus its counters."""
        J = j1 - j0
        js = np.arange(j0, j1, dtype=np.int64)
        phi = np.ascontiguousarray(phi0s, np.complex128)
        counts = np.zeros(5, np.int64)
        _check(_lib.gf_memcpy(self.basis, js.ctypes.data, js.nbytes, H2D, None))
        _check(_lib.gf_memcpy(self.phi0, phi.ctypes.data, phi.nbytes, H2D, None))
        _check(_lib.gf_hess_plan_eval(self.h, J, self.basis, None, self.phi0, self.out, counts.ctypes.data, None))
        _check(_lib.gf_hess_plan_slot_outputs(self.h, J, self.slots, None))
        rec = np.empty(self.rec)
        dacc = np.empty((self.n, 4, 4), np.complex128)
        _check(_lib.gf_memcpy(rec.ctypes.data, self.out, rec.nbytes, D2H, None))
        _check(_lib.gf_memcpy(dacc.ctypes.data, self.slots, dacc.nbytes, D2H, None))
        _check(_lib.gf_stream_sync(None))
        nlog32 = self.rec - 2 - 2 * self.R * self.A * self.A
        blocks = rec[2 + nlog32:].view(np.complex128).reshape(self.R, self.A, self.A).copy()
        return complex(rec[0], rec[1]), dacc, blocks, counts
