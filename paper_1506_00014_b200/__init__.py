"""B200-native log-polar Radon transform R and back-projection R# (arXiv 1506.00014).

Host mirror of the reference's lp_ops interface over the C ABI in
``include/lpradon_gpu.h``; the compute runs in hand-written sm_100a kernels
(``csrc/``). See DESIGN.md.
"""
from .lp_ops import (  # noqa: F401
    Geometry,
    RadonPlan,
    adjoint_gap,
    apply_filter,
    em_run,
    fast_backprojection,
    fbp,
    fast_radon,
    inner_image,
    inner_sinogram,
    lp_convolve,
    radon_backproject,
    radon_transpose,
    sampling_plan,
    sensitivity_image,
    set_spectrum_cache,
    spectrum_cache_counters,
    smooth_n_rho,
    zeta_bp_spectrum,
    zeta_spectrum,
)
