"""ctypes binding of libpftg.so (include/pftg.h).

The library is built in-tree (``make -C paper_2408_03532_b200/csrc``, or
``__graft_entry__.build()``). There is no fallback: if the shared object is
missing or no sm_100 GPU is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
# PFTG_LIB_PATH: an alternative build (e.g. the -DPFTG_PROFILING library of tools/)
LIB_PATH = Path(os.environ["PFTG_LIB_PATH"]) if os.environ.get("PFTG_LIB_PATH") else HERE / "libpftg.so"

PFTG_OK, PFTG_EINVAL, PFTG_ELOGIC, PFTG_ERANGE, PFTG_ERUNTIME, PFTG_ECUDA = range(6)
PFTG_C64, PFTG_C128 = 0, 1

# Every symbol include/pftg.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "pftg_version", "pftg_last_error", "pftg_device_ok", "pftg_profile_begin", "pftg_profile_end", "pftg_profile_mode",
    "pftg_table_load", "pftg_table_free", "pftg_table_min_degree",
    "pftg_best_approx", "pftg_table_compute", "pftg_table_save", "pftg_table_info", "pftg_table_record",
    "pftg_measurements_save", "pftg_measurements_info", "pftg_measurements_read",
    "pftg_plan_2d", "pftg_plan_from_tables", "pftg_plan_load", "pftg_plan_save", "pftg_plan_free", "pftg_plan_info",
    "pftg_plan_tables",
    "pftg_apply_2d_dev", "pftg_adjoint_2d_dev", "pftg_apply_2d_host", "pftg_adjoint_2d_host", "pftg_fwd_adj_2d_host",
    "pftg_apply_2d_host_multi", "pftg_adjoint_2d_host_multi", "pftg_fwd_adj_2d_host_multi",
    "pftg_band_residual_dev",
    "pftg_fft2_dev", "pftg_fft2_host", "pftg_project_modulus_dev", "pftg_crop_centered_dev",
    "pftg_window_slice_dev", "pftg_set_window_dev", "pftg_pie_object_update_dev",
    "pftg_epie_probe_update_dev", "pftg_evaluate_dev",
    "pftg_simulate_dev", "pftg_add_poisson_noise_dev", "pftg_fill_metrics_dev",
    "pftg_plan_1d", "pftg_plan1d_from_tables", "pftg_plan1d_load", "pftg_plan1d_save", "pftg_plan1d_info",
    "pftg_plan1d_tables", "pftg_plan1d_free", "pftg_apply_1d_dev", "pftg_apply_1d_host",
    "pftg_solver_create", "pftg_solver_run", "pftg_solver_trace", "pftg_solver_result",
    "pftg_solver_device_state", "pftg_solver_free",
)


class CudaError(RuntimeError):
    """A CUDA failure inside libpftg (no device, launch error, fault)."""


class SolverConfigC(C.Structure):
    _fields_ = [
        ("pft_sweeps", C.c_int), ("fft_sweeps", C.c_int),
        ("beta", C.c_double), ("gamma", C.c_double), ("beta_pft", C.c_double),
        ("gamma_pft", C.c_double), ("eps_pft", C.c_double), ("tol", C.c_double),
        ("mt1", C.c_int64), ("mt2", C.c_int64), ("p1", C.c_int64), ("p2", C.c_int64),
        ("blind", C.c_int), ("shuffled", C.c_int), ("seed", C.c_uint64),
        ("objective_every", C.c_int),
        ("tv_lambda_mag", C.c_double), ("tv_lambda_phase", C.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"libpftg.so not built ({LIB_PATH}); run `make -C paper_2408_03532_b200/csrc` "
            "or __graft_entry__.build(). There is no CPU fallback.")
    L = C.CDLL(str(LIB_PATH))
    vp, sz, dp, i64p = C.c_void_p, C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_int64)
    L.pftg_last_error.restype = C.c_char_p
    L.pftg_profile_end.argtypes = [dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.pftg_table_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.pftg_table_free.argtypes = [vp]
    L.pftg_table_free.restype = None
    L.pftg_table_min_degree.argtypes = [vp, C.c_double, C.c_double, C.POINTER(C.c_int)]
    L.pftg_plan_2d.argtypes = [vp, sz, sz, sz, sz, sz, sz, C.c_double, C.POINTER(vp)]
    L.pftg_plan_from_tables.argtypes = [sz, sz, sz, C.c_int, dp, dp, sz, sz, sz, C.c_int, dp, dp,
                                        C.c_double, C.POINTER(vp)]
    L.pftg_plan_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.pftg_plan_save.argtypes = [vp, C.c_char_p]
    L.pftg_plan_free.argtypes = [vp]
    L.pftg_plan_free.restype = None
    L.pftg_plan_info.argtypes = [vp, i64p]
    L.pftg_plan_tables.argtypes = [vp, C.c_int, dp, dp]
    L.pftg_apply_2d_dev.argtypes = [vp, C.c_int, vp, vp, sz, vp]
    L.pftg_adjoint_2d_dev.argtypes = [vp, C.c_int, vp, vp, sz, vp]
    L.pftg_apply_2d_host.argtypes = [vp, C.c_int, vp, vp, sz]
    L.pftg_adjoint_2d_host.argtypes = [vp, C.c_int, vp, vp, sz]
    L.pftg_fwd_adj_2d_host.argtypes = [vp, C.c_int, vp, vp, vp, sz]
    ip = C.POINTER(C.c_int)
    L.pftg_apply_2d_host_multi.argtypes = [vp, C.c_int, vp, vp, sz, ip, C.c_int]
    L.pftg_adjoint_2d_host_multi.argtypes = [vp, C.c_int, vp, vp, sz, ip, C.c_int]
    L.pftg_fwd_adj_2d_host_multi.argtypes = [vp, C.c_int, vp, vp, vp, sz, ip, C.c_int]
    L.pftg_band_residual_dev.argtypes = [vp, C.c_int, vp, vp, vp, sz, vp]
    L.pftg_fft2_dev.argtypes = [C.c_int, vp, vp, sz, sz, sz, C.c_int, vp]
    L.pftg_fft2_host.argtypes = [C.c_int, vp, vp, sz, sz, sz, C.c_int]
    L.pftg_project_modulus_dev.argtypes = [C.c_int, vp, vp, vp, sz, sz, sz, vp]
    L.pftg_crop_centered_dev.argtypes = [C.c_int, vp, vp, sz, sz, sz, sz, sz, vp]
    L.pftg_window_slice_dev.argtypes = [C.c_int, vp, sz, sz, vp, sz, sz, i64p, sz, vp]
    L.pftg_set_window_dev.argtypes = [C.c_int, vp, sz, sz, vp, sz, sz, C.c_int64, C.c_int64, vp]
    L.pftg_pie_object_update_dev.argtypes = [C.c_int, vp, vp, vp, sz, C.c_double, vp]
    L.pftg_epie_probe_update_dev.argtypes = [C.c_int, vp, vp, vp, sz, C.c_double, C.c_int, vp]
    L.pftg_evaluate_dev.argtypes = [C.c_int, vp, sz, sz, vp, sz, sz, i64p, sz, sz, sz, vp, vp, vp,
                                    dp, dp, vp]
    L.pftg_simulate_dev.argtypes = [C.c_int, vp, sz, sz, vp, sz, sz, i64p, sz, vp, vp]
    L.pftg_add_poisson_noise_dev.argtypes = [C.c_int, vp, sz, C.c_double, C.c_uint64, vp]
    L.pftg_fill_metrics_dev.argtypes = [C.c_int, vp, sz, vp, sz, sz, sz, dp, vp]
    L.pftg_best_approx.argtypes = [C.c_int, C.c_double, dp, dp]
    L.pftg_table_compute.argtypes = [dp, C.c_int, C.c_int, C.POINTER(vp)]
    L.pftg_table_save.argtypes = [vp, C.c_char_p]
    L.pftg_table_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.pftg_table_record.argtypes = [vp, C.c_int, dp, C.POINTER(C.c_int), dp, dp, dp]
    L.pftg_measurements_save.argtypes = [C.c_char_p, sz, sz, sz, dp, sz, sz, dp, C.c_double, C.c_uint64]
    L.pftg_measurements_info.argtypes = [C.c_char_p, i64p, dp, C.POINTER(C.c_uint64)]
    L.pftg_measurements_read.argtypes = [C.c_char_p, C.c_int, vp, vp]
    L.pftg_plan_1d.argtypes = [vp, sz, sz, sz, C.c_double, C.POINTER(vp)]
    L.pftg_plan1d_from_tables.argtypes = [sz, sz, sz, C.c_int, dp, dp, C.c_double, C.POINTER(vp)]
    L.pftg_plan1d_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.pftg_plan1d_save.argtypes = [vp, C.c_char_p]
    L.pftg_plan1d_info.argtypes = [vp, i64p]
    L.pftg_plan1d_tables.argtypes = [vp, dp, dp]
    L.pftg_plan1d_free.argtypes = [vp]
    L.pftg_plan1d_free.restype = None
    L.pftg_apply_1d_dev.argtypes = [vp, C.c_int, vp, vp, sz, vp]
    L.pftg_apply_1d_host.argtypes = [vp, C.c_int, vp, vp, sz]
    L.pftg_solver_create.argtypes = [C.c_int, vp, sz, sz, vp, sz, sz, i64p, sz, vp,
                                     C.POINTER(SolverConfigC), vp, C.POINTER(vp)]
    L.pftg_solver_run.argtypes = [vp, C.c_int]
    L.pftg_solver_trace.argtypes = [vp, dp, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.pftg_solver_result.argtypes = [vp, vp, vp]
    L.pftg_solver_device_state.argtypes = [vp, C.POINTER(vp), C.POINTER(vp)]
    L.pftg_solver_free.argtypes = [vp]
    L.pftg_solver_free.restype = None
    _lib = L
    return L


KERNEL_NAMES = ("pft_rows_fwd", "pft_cols_fwd", "pft_cols_adj", "pft_rows_adj", "fft_rows",
                "fft_cols")


class KernelProfile:
    """Context manager over pftg_profile_begin/end: per-kernel CUDA-event time.
    isolate=True spins the stream before each launch so the events time the
    kernel alone (replays outside a timed region); count_only=True records no
    events, only launch counts (safe inside a timed region)."""

    def __init__(self, isolate=False, count_only=False):
        self.mode = 2 if count_only else (1 if isolate else 0)

    def __enter__(self):
        check(lib().pftg_profile_mode(self.mode))
        check(lib().pftg_profile_begin())
        return self

    def __exit__(self, *exc):
        ms = (C.c_double * len(KERNEL_NAMES))()
        cnt = (C.c_int * len(KERNEL_NAMES))()
        launches = (C.c_int * len(KERNEL_NAMES))()
        check(lib().pftg_profile_end(ms, cnt, launches))
        check(lib().pftg_profile_mode(0))
        self.ms = {KERNEL_NAMES[k]: ms[k] for k in range(len(KERNEL_NAMES))}
        self.count = {KERNEL_NAMES[k]: cnt[k] for k in range(len(KERNEL_NAMES))}
        self.launches = {KERNEL_NAMES[k]: launches[k] for k in range(len(KERNEL_NAMES))}
        return False


def check(rc: int) -> None:
    """Map a pftg status onto the Python analogue of the reference's exception."""
    if rc == PFTG_OK:
        return
    msg = lib().pftg_last_error().decode(errors="replace")
    if rc == PFTG_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == PFTG_ERANGE:
        raise IndexError(msg)          # std::out_of_range
    if rc == PFTG_ELOGIC:
        raise RuntimeError(msg)        # std::logic_error
    if rc == PFTG_ECUDA:
        raise CudaError(msg)
    raise OSError(msg)                 # std::runtime_error (I/O, format)
