"""stratcox-b200: B200-native (sm_100a) stratified Cox partial likelihood and
L1 cyclic coordinate descent — the hot path of arXiv 2310.16238 behind the
reference ``stratcox`` API.

The compute runs in ``libstratcox_b200.so`` (csrc/, C-ABI in
include/stratcox_b200.h); this package is the host-side mirror of the
reference interface.
"""
from .stratcox import (  # noqa: F401
    CoefficientState,
    CudaError,
    DeviceDesign,
    ExecutionConfig,
    FitResult,
    GradHess,
    InternalError,
    NumericError,
    OptimizerConfig,
    PenaltySpec,
    ProposedStep,
    SortedDesign,
    StratcoxError,
    TrustOutcome,
    ValidationError,
    CvResult,
    SurvivalDataset,
    apply_trust_region,
    build_design,
    build_lowered_design,
    ccd_fit,
    fold_assignment,
    kfold_select_gamma,
    lower_time_varying,
    default_gamma_grid,
    device_count,
    gamma_max,
    gradient_hessian,
    l1_coordinate_update,
    coordinate_update,
    log_partial_likelihood,
    make_state,
    naive_gradient_hessian,
    naive_log_partial_likelihood,
    newton_step,
    refresh_xbeta,
    risk_suffix_gradient_hessian,
    segmented_inclusive_scan,
    state_from_arrays,
    update_xbeta,
    upload,
)

__version__ = "0.1.0"
