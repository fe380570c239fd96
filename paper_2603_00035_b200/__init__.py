"""B200-native differentiable Randers eikonal hot path (arXiv 2603.00035).

The product is the CUDA library ``librfk.so`` behind the C ABI in
``include/rfk.h``; :mod:`.api` mirrors the reference's
``proj/include/randers`` API on top of it.
"""
from .api import (  # noqa: F401
    Context, CudaError, DimensionMismatch, Error, InconsistentFixedPoint, InvalidArgument,
    NoDevice, NotConverged, Objective, Records, SolveReport, ZeroDimension, backward, best_candidate, best_candidates,
    context, drift_norm_sq, identify_stencils, jacobi_iteration_budget, jacobian_entries,
    loss_grad_mse, node_update, objective_and_grad, param_gradients, project_drift, project_drift_vjp, project_spd,
    project_spd_vjp, project_vjp, solve, solve_f32, backward_f32, Projection, solve_projected, backward_projected,
    solve_adjoint, solve_from_values, solve_jacobi, two_point_update, NonSpdInput, DivergedLoss,
)
from .inverse import (  # noqa: F401
    AdamState, InverseConfig, OptimizerKind, Parameterization, RecoveryResult, TvVariant, adam_step,
    clip_global_norm, generate_observations, gd_step, multi_source_recover, MultiSourceRow, objective, recover, relative_error, tikhonov_value_grad,
    tv_value_grad,
)
