"""B200-native (sm_100a) fast Partial Fourier Transform and PFT-warm-started
ePIE -- a drop-in for the PFT / ePIE hot path of the reference library
``proj/core`` (arXiv:2408.03532). The compute path is libpftg.so (CUDA kernels
behind the C-ABI in include/pftg.h); this package is the Python host mirror of
the reference's operator API. There is no CPU fallback.
"""
from ._lib import CudaError, LIB_PATH  # noqa: F401
from .pft import (  # noqa: F401
    DEFAULT_TABLE, PftPlan1D, PftPlan2D, ScopeTable, band_residual, crop_centered, fast_fft2,
    fast_ifft2, best_approx, pft_adjoint_2d, pft_fwd_adj_2d, pft_apply_1d, pft_apply_2d, pft_plan_1d, pft_plan_2d)
from .solver import (  # noqa: F401
    ReconResult, Solver, SolverConfig, epie_probe_update, evaluate, hybrid_solve,
    objective_value, pie_object_update, project_modulus, set_window, solve_epie, solve_pie,
    window_slice)
from .simulate import (add_poisson_noise, build_cropped, load_measurements, photon_scale,  # noqa: E402
                       save_measurements, simulate)  # noqa: F401,E402
from .metrics import Metrics, fill_metrics, relative_error, relative_error_aligned  # noqa: F401,E402
