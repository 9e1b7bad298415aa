"""ctypes binding of libgfcuda.so (the C ABI declared in include/gatefit_b200.h).

There is no fallback: if the shared library is missing the import fails
loudly, and every compute entry point needs a CUDA device.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GF_LIB_PATH") or os.path.join(HERE, "libgfcuda.so")

GF_OK, GF_EINVAL, GF_ENONFINITE, GF_ECUDA, GF_ENOMEM = range(5)
GF_VALUE, GF_GRAD, GF_HVP = 1, 2, 4

# every symbol of include/gatefit_b200.h (checked by tests/test_abi.py)
EXPORTS = (
    "gf_last_error",
    "gf_abi_version",
    "gf_apply_gate",
    "gf_apply_gate_1q",
    "gf_apply_gate_sector_c1q",
    "gf_hole_contract",
    "gf_hole_apply",
    "gf_apply_gate_to_array",
    "gf_hole_contract_array",
    "gf_sector_unrank",
    "gf_sector_rank",
    "gf_orbit_canon",
    "gf_sector_orbit_mark",
    "gf_plan_create",
    "gf_plan_set_gates",
    "gf_plan_set_directions",
    "gf_plan_set_directions_multi",
    "gf_plan_eval",
    "gf_plan_slot_outputs",
    "gf_plan_last_launches",
    "gf_plan_set_profiling",
    "gf_plan_phase_times",
    "gf_plan_describe",
    "gf_plan_live_fraction",
    "gf_plan_first_reverse_pass",
    "gf_plan_layout",
    "gf_plan_destroy",
    "gf_hess_plan_create",
    "gf_hess_plan_set_gates",
    "gf_hess_plan_eval",
    "gf_hess_plan_slot_outputs",
    "gf_hess_plan_last_launches",
    "gf_hess_plan_destroy",
    "gf_cheb_step",
    "gf_hamiltonian_apply",
    "gf_nb_cheb_step",
    "gf_nb_scatter",
    "gf_nb_rank",
    "gf_nb_gather",
    "gf_nb_block_matrix",
    "gf_peak_fp64",
    "gf_check_finite",
    "gf_set_device",
    "gf_malloc",
    "gf_free",
    "gf_memcpy",
    "gf_stream_sync",
)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')"
    )

lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64

lib.gf_last_error.restype = ctypes.c_char_p
lib.gf_abi_version.restype = _i
lib.gf_plan_last_launches.restype = _i64
lib.gf_plan_last_launches.argtypes = [_vp]
lib.gf_hess_plan_last_launches.restype = _i64
lib.gf_hess_plan_last_launches.argtypes = [_vp]
for _name, _args in {
    "gf_apply_gate": [_vp, _vp, _i, _i, _i, _vp, _i, _i64, _vp],
    "gf_apply_gate_sector_c1q": [_vp, _vp, _i, _i, _i, _vp, _i64, _vp],
    "gf_apply_gate_1q": [_vp, _vp, _i, _i, _vp, _i64, _vp],
    "gf_hole_contract": [_vp, _vp, _i, _i, _i, _i64, _vp, _vp],
    "gf_hole_apply": [_vp, _vp, _i, _i, _i, _vp, _i, _vp],
    "gf_apply_gate_to_array": [_vp, _vp, _i, _i, _i, _i, _vp, _i, _vp],
    "gf_hole_contract_array": [_vp, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp],
    "gf_sector_unrank": [_vp, _i64, _i, _vp, _vp],
    "gf_sector_rank": [_vp, _i64, _vp, _vp],
    "gf_orbit_canon": [_vp, _i64, _i, _vp, _vp, _vp],
    "gf_sector_orbit_mark": [_i64, _i64, _i, _i, _vp, _vp],
    "gf_plan_create": [ctypes.POINTER(_vp), _i, _i, _i, _vp, _vp, _vp, _i, _i64, _i],
    "gf_plan_set_gates": [_vp, _vp],
    "gf_plan_set_directions": [_vp, _vp],
    "gf_plan_set_directions_multi": [_vp, _i, _vp],
    "gf_plan_eval": [_vp, _i, _i64, _vp, _vp, _vp, _vp, _vp],
    "gf_plan_slot_outputs": [_vp, _i64, _vp, _vp, _vp],
    "gf_plan_destroy": [_vp],
    "gf_hess_plan_create": [ctypes.POINTER(_vp), _i, _i, _vp, _vp, _vp, _i, _vp, _i, _vp, _i64, _vp, _vp, _vp, _vp,
                            _vp, _vp, _i64, _i],
    "gf_hess_plan_set_gates": [_vp, _vp, _i],
    "gf_hess_plan_eval": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "gf_hess_plan_slot_outputs": [_vp, _i64, _vp, _vp],
    "gf_hess_plan_destroy": [_vp],
    "gf_plan_describe": [_vp, _vp, _vp, _vp, _vp, _vp],
    "gf_plan_live_fraction": [_vp, _vp],
    "gf_plan_first_reverse_pass": [_vp, _vp, _vp, _vp, _vp],
    "gf_plan_layout": [_i, _i, _i, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp],
    "gf_plan_set_profiling": [_vp, _i],
    "gf_plan_phase_times": [_vp, _vp, _vp],
    "gf_cheb_step": [_vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i, ctypes.c_double, ctypes.c_double,
                     ctypes.c_double, ctypes.c_double, _i64, _i, _vp],
    "gf_hamiltonian_apply": [_vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _i64, _vp],
    "gf_peak_fp64": [_i, _i, _i, _vp, _vp, _vp],
    "gf_nb_cheb_step": [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                        ctypes.c_double, _i64, _vp],
    "gf_nb_scatter": [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _i, _i, _vp],
    "gf_nb_rank": [_vp, _vp, _i64, _vp, _i, _vp],
    "gf_nb_block_matrix": [_vp, _vp, _i, _vp, _vp, _i, _vp, _i, ctypes.c_double, ctypes.c_double, _vp, _vp],
    "gf_nb_gather": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i, _vp, _i64, _vp],
    "gf_check_finite": [_vp, _i64, _vp],
    "gf_set_device": [_i],
    "gf_malloc": [ctypes.POINTER(_vp), _i64],
    "gf_free": [_vp],
    "gf_memcpy": [_vp, _vp, _i64, _i, _vp],
    "gf_stream_sync": [_vp],
}.items():
    getattr(lib, _name).argtypes = _args
    getattr(lib, _name).restype = _i


class EngineError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map a gf_status to the reference's exception classes."""
    if rc == GF_OK:
        return
    msg = (lib.gf_last_error() or b"").decode(errors="replace")
    if rc == GF_EINVAL:
        raise ValueError(msg)
    if rc == GF_ENONFINITE:
        raise FloatingPointError(msg)
    if rc == GF_ENOMEM:
        raise MemoryError(msg)
    raise EngineError(msg)


def ptr(t) -> int | None:
    """Raw device / host address of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None) -> int | None:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
