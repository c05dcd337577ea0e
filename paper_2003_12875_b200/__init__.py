"""B200-native batched PDF-graph evaluation + unbinned NLL (arXiv 2003.12875 hot path).

The product is the C-ABI library ``lib/libffit_b200.so`` (CUDA sm_100a kernels +
C++ host engine, sources in ``csrc/``, header ``include/ffit_b200.h``); this
package is its Python mirror of the reference interface.
"""
from ._lib import LIB_PATH, build, lib  # noqa: F401
from .ffit import (  # noqa: F401
    DataSet, EvalMode, FfitError, FitResult, Model, NllValue, ShardGroup, eval_batch, eval_batch_device, expr_eval, expression_jit,
    expression_jit_source, expression_jit_status, fit_gradient, fit_to, grad_spec_source, last_grad_jit,
    last_launch_jit, last_launch_cached, plan_spec_min_work, plan_spec_source,
    fp64_issue_probe, fp64_peak, kernel_launches, kernel_timer, kernel_timer_read, last_launch, nll, nll_c, nll_points,
    nll_points_device, nll_grad, nll_grad_finish, nll_grad_partial, grad_slot_count,
    nll_points_partial, normalization, device_normalization, device_normalization_enabled, device_normalization_launches,
    set_device_normalization, probabilities, read_soa_host, sample_host, write_soa)
