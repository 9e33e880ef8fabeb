"""ctypes binding of ``libsdcsw.so`` (declared in ``include/sdcsw.h``).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, :func:`lib` raises :class:`DeviceError` immediately.
"""

import ctypes
import os

from .errors import DeviceError, DivergenceError, ParameterError

LIB_PATH = os.environ.get("SDCSW_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libsdcsw.so")  # env: experiment builds only

SDCSW_OK, SDCSW_ERR_PARAM, SDCSW_ERR_CUDA, SDCSW_ERR_STATE, SDCSW_ERR_DIVERGED, SDCSW_ERR_PEER = range(6)
IPC_HANDLE_BYTES = 64  # SDCSW_IPC_HANDLE_BYTES
SWEEP_HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int)  # sdcsw_sweep_hook
COMM_ID_BYTES = 128  # SDCSW_COMM_ID_BYTES

EXPORTS = (
    "sdcsw_plan_create",
    "sdcsw_plan_create_planar",
    "sdcsw_plan_destroy",
    "sdcsw_f_expl",
    "sdcsw_f_impl",
    "sdcsw_implicit_solve",
    "sdcsw_sweep_nodes",
    "sdcsw_sweep_nodes_residual",
    "sdcsw_final_node",
    "sdcsw_serial_sweep",
    "sdcsw_stepper_create",
    "sdcsw_stepper_create_ensemble",
    "sdcsw_stepper_destroy",
    "sdcsw_stepper_run",
    "sdcsw_stepper_diverged",
    "sdcsw_stepper_reset",
    "sdcsw_stepper_launches_per_step",
    "sdcsw_stepper_set_option",
    "sdcsw_stepper_profile",
    "sdcsw_stepper_step_hooked",
    "sdcsw_stepper_sweep_state",
    "sdcsw_stepper_storage",
    "sdcsw_check_finite",
    "sdcsw_axpy",
    "sdcsw_transform_stage",
    "sdcsw_workspace",
    "sdcsw_plan_transform_kind",
    "sdcsw_plan_set_split",
    "sdcsw_split_info",
    "sdcsw_split_f_expl_begin",
    "sdcsw_split_f_expl_end",
    "sdcsw_exchange_create",
    "sdcsw_exchange_create_split",
    "sdcsw_exchange_ipc_handle",
    "sdcsw_exchange_open_peers",
    "sdcsw_exchange_base",
    "sdcsw_exchange_attach_peer",
    "sdcsw_exchange_phase",
    "sdcsw_exchange_post",
    "sdcsw_exchange_run",
    "sdcsw_exchange_set_option",
    "sdcsw_exchange_info",
    "sdcsw_exchange_diverged",
    "sdcsw_exchange_reset",
    "sdcsw_exchange_destroy",
    "sdcsw_comm_unique_id",
    "sdcsw_comm_create",
    "sdcsw_comm_init_all",
    "sdcsw_comm_split",
    "sdcsw_comm_info",
    "sdcsw_allgather_rhs",
    "sdcsw_comm_destroy",
    "sdcsw_nccl_version",
    "sdcsw_guard_check",
    "sdcsw_guard_selftest",
    "sdcsw_last_error",
    "sdcsw_version",
)


class Config(ctypes.Structure):
    _fields_ = [
        ("trunc", ctypes.c_int),
        ("nlat", ctypes.c_int),
        ("nlon", ctypes.c_int),
        ("max_batch", ctypes.c_int),
        ("radius", ctypes.c_double),
        ("omega", ctypes.c_double),
        ("phibar", ctypes.c_double),
    ]


class PlanarConfig(ctypes.Structure):
    _fields_ = [
        ("n_grid", ctypes.c_int),
        ("max_batch", ctypes.c_int),
        ("domain_length", ctypes.c_double),
        ("mean_geopotential", ctypes.c_double),
        ("coriolis", ctypes.c_double),
        ("hyperviscosity", ctypes.c_double),
    ]


_LIB = None
_p = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)

_SIGS = {
    "sdcsw_plan_create": [_i, ctypes.POINTER(Config), _dp, _dp, _dp, _dp, _ip, _ip, _ip, _dp,
                          ctypes.POINTER(_p)],
    "sdcsw_plan_create_planar": [_i, ctypes.POINTER(PlanarConfig), _dp, _dp, _dp,
                                 ctypes.POINTER(_p)],
    "sdcsw_plan_destroy": [_p],
    "sdcsw_f_expl": [_p, _p, _p, _i, _p],
    "sdcsw_f_impl": [_p, _p, _p, _i, _p],
    "sdcsw_implicit_solve": [_p, _dp, _p, _p, _i, _p],
    "sdcsw_sweep_nodes": [_p, _i, _i, _i, _dp, _p, _p, _ll, _p, _ll, _i, _p, _p, _p],
    "sdcsw_sweep_nodes_residual": [_p, _i, _i, _i, _dp, _p, _p, _ll, _p, _ll, _i, _p, _p, _p, _p,
                                   _p],
    "sdcsw_final_node": [_p, _i, _dp, _p, _p, _ll, _p, _ll, _i, _p, _p],
    "sdcsw_serial_sweep": [_p, _i, _dp, _p, _p, _ll, _p, _ll, _i, _p, _p, _p, _p, _p],
    "sdcsw_stepper_create": [_p, _i, _i, _i, _dp, _i, ctypes.POINTER(_p)],
    "sdcsw_stepper_create_ensemble": [_p, _i, _i, _i, _i, _dp, _i, ctypes.POINTER(_p)],
    "sdcsw_stepper_destroy": [_p],
    "sdcsw_stepper_run": [_p, _p, _i, _i, _p],
    "sdcsw_stepper_diverged": [_p, _ip],
    "sdcsw_stepper_reset": [_p, _p],
    "sdcsw_stepper_launches_per_step": [_p, _ip],
    "sdcsw_stepper_set_option": [_p, _i, _i],
    "sdcsw_stepper_profile": [_p, _p, _dp, _i, _p],
    "sdcsw_stepper_step_hooked": [_p, _p, _p, _p, _dp, _i, _p],
    "sdcsw_stepper_sweep_state": [_p, _i, ctypes.POINTER(_p), ctypes.POINTER(_p), ctypes.POINTER(_p)],
    "sdcsw_stepper_storage": [_p, ctypes.POINTER(_ll), ctypes.POINTER(_ll)],
    "sdcsw_check_finite": [_p, _ll, _p, _p],
    "sdcsw_axpy": [_ll, _p, ctypes.c_double, _p, _p, _p],
    "sdcsw_transform_stage": [_p, _i, _p, _p, _i, _p],
    "sdcsw_workspace": [_p, _i, ctypes.POINTER(_p), ctypes.POINTER(_ll)],
    "sdcsw_plan_transform_kind": [_p, _ip, _ip],
    "sdcsw_plan_set_split": [_p, _i, _i, _p, _ll],
    "sdcsw_split_info": [_p, _ip, _ip, _ip],
    "sdcsw_split_f_expl_begin": [_p, _p, _i, _p],
    "sdcsw_split_f_expl_end": [_p, _p, _i, _p],
    "sdcsw_exchange_create": [_p, _i, _i, _dp, _i, _i, _i, ctypes.POINTER(_p)],
    "sdcsw_exchange_create_split": [_p, _i, _i, _dp, _i, _i, _i, _i, ctypes.POINTER(_p)],
    "sdcsw_exchange_ipc_handle": [_p, _p, _i],
    "sdcsw_exchange_open_peers": [_p, _p, _i],
    "sdcsw_exchange_base": [_p, ctypes.POINTER(_p)],
    "sdcsw_exchange_attach_peer": [_p, _i, _p],
    "sdcsw_exchange_phase": [_p, _p, _i, _p],
    "sdcsw_exchange_post": [_p, _i, _i, _p],
    "sdcsw_exchange_run": [_p, _p, _i, _i, _p],
    "sdcsw_exchange_set_option": [_p, _i, _i],
    "sdcsw_exchange_info": [_p, _ip, _ip, _ip],
    "sdcsw_exchange_diverged": [_p, _ip],
    "sdcsw_exchange_reset": [_p, _p],
    "sdcsw_exchange_destroy": [_p],
    "sdcsw_comm_unique_id": [_p, _i],
    "sdcsw_comm_create": [_p, _i, _i, _i, _i, ctypes.POINTER(_p)],
    "sdcsw_comm_init_all": [_i, _ip, ctypes.POINTER(_p)],
    "sdcsw_comm_split": [_p, _i, _i, ctypes.POINTER(_p)],
    "sdcsw_comm_info": [_p, _ip, _ip],
    "sdcsw_allgather_rhs": [_p, _p, _p, _ll, _p],
    "sdcsw_comm_destroy": [_p],
    "sdcsw_nccl_version": [],
    "sdcsw_guard_check": [ctypes.POINTER(ctypes.c_longlong), _ip],
    "sdcsw_guard_selftest": [],
    "sdcsw_last_error": [],
    "sdcsw_version": [],
}


def load(path=LIB_PATH):
    """Load the library and bind every exported symbol (no GPU needed)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise DeviceError(
            f"{path} is not built; run `python -m paper_2403_20135_b200.build` "
            "(the CUDA path has no CPU fallback)"
        )
    lib_ = ctypes.CDLL(path)
    partial = os.environ.get("SDCSW_LIB_PARTIAL") == "1"  # experiment builds of older sources
    for name, args in _SIGS.items():
        if partial and not hasattr(lib_, name):
            continue
        fn = getattr(lib_, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name == "sdcsw_last_error" else ctypes.c_int
    _LIB = lib_
    return lib_


def lib():
    """The library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the sdcsw path runs only on a B200 (sm_100a)")
    return load()


def check(status, what="sdcsw"):
    if status == SDCSW_OK:
        return
    msg = (_LIB.sdcsw_last_error() or b"").decode() if _LIB is not None else ""
    if status == SDCSW_ERR_PARAM:
        raise ParameterError(f"{what}: {msg}")
    if status == SDCSW_ERR_DIVERGED:
        raise DivergenceError(f"{what}: {msg}", step_index=-1)
    raise DeviceError(f"{what}: {msg}", code=status)


def dptr(arr):
    """ctypes double* of a C-contiguous float64 numpy array."""
    return arr.ctypes.data_as(_dp)


def iptr(arr):
    return arr.ctypes.data_as(_ip)
