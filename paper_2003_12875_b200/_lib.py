"""Loads the product library (lib/libffit_b200.so) and declares its C ABI.

There is no fallback: if the shared library is missing the import fails loudly,
and if no CUDA device is usable every evaluation call returns FFIT_ERR_NUMERIC.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# FFB_LIB_VARIANT=<tag> loads lib/ab/libffit_b200_<tag>.so instead (A/B builds of the
# same sources with different -D switches, csrc/Makefile `ab` target)
_variant = os.environ.get("FFB_LIB_VARIANT")
LIB_PATH = (os.path.join(HERE, "lib", "ab", f"libffit_b200_{_variant}.so") if _variant
            else os.path.join(HERE, "lib", "libffit_b200.so"))
CSRC = os.path.join(HERE, "csrc")

D = ctypes.c_double
DP = ctypes.POINTER(ctypes.c_double)
LL = ctypes.c_longlong
LLP = ctypes.POINTER(ctypes.c_longlong)
ULL = ctypes.c_ulonglong
ULLP = ctypes.POINTER(ctypes.c_ulonglong)
VP = ctypes.c_void_p
CP = ctypes.c_char_p
I = ctypes.c_int
IP = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); every symbol include/ffit_b200.h declares
SIGNATURES = {
    "ffit_last_error": (CP, []),
    "ffit_model_load": (I, [CP, ctypes.POINTER(VP)]),
    "ffit_model_parse": (I, [CP, ctypes.POINTER(VP)]),
    "ffit_model_free": (None, [VP]),
    "ffit_model_observable": (CP, [VP]),
    "ffit_model_observable_range": (I, [VP, DP, DP]),
    "ffit_model_param_count": (I, [VP]),
    "ffit_model_param_name": (CP, [VP, I]),
    "ffit_model_param_is_constant": (I, [VP, CP, IP]),
    "ffit_model_get_param": (I, [VP, CP, DP, DP]),
    "ffit_model_set_param": (I, [VP, CP, D]),
    "ffit_dataset_read_csv": (I, [VP, CP, ctypes.POINTER(VP), ctypes.POINTER(ctypes.c_long)]),
    "ffit_dataset_write_csv": (I, [VP, CP]),
    "ffit_dataset_rows": (ctypes.c_long, [VP]),
    "ffit_dataset_free": (None, [VP]),
    "ffit_sample": (I, [VP, ctypes.c_long, ULL, ctypes.POINTER(VP), DP]),
    "ffit_nll": (I, [VP, VP, I, DP, ULLP]),
    "ffit_probabilities": (I, [VP, VP, I, DP]),
    "ffit_fit": (I, [VP, VP, I, D, ctypes.c_long, ctypes.POINTER(VP)]),
    "ffit_result_converged": (I, [VP]),
    "ffit_result_nll": (D, [VP]),
    "ffit_result_nll_calls": (ULL, [VP]),
    "ffit_result_wall_seconds": (D, [VP]),
    "ffit_result_uncertainties_valid": (I, [VP]),
    "ffit_result_param_count": (I, [VP]),
    "ffit_result_param_name": (CP, [VP, I]),
    "ffit_result_param_value": (D, [VP, I]),
    "ffit_result_param_uncertainty": (D, [VP, I]),
    "ffit_result_free": (None, [VP]),
    "ffcu_dataset_from_host": (I, [ctypes.POINTER(CP), ctypes.POINTER(DP), I, LL, ctypes.POINTER(VP)]),
    "ffcu_dataset_from_device": (I, [ctypes.POINTER(CP), ctypes.POINTER(VP), I, LL, I, ctypes.POINTER(VP)]),
    "ffcu_dataset_copy_from_host": (I, [VP, ctypes.POINTER(DP)]),
    "ffcu_dataset_copy_from_host_async": (I, [VP, ctypes.POINTER(DP), VP]),
    "ffcu_dataset_slice": (I, [VP, LL, LL, ctypes.POINTER(VP)]),
    "ffcu_dataset_ncols": (I, [VP]),
    "ffcu_dataset_column_name": (CP, [VP, I]),
    "ffcu_dataset_download": (I, [VP, I, DP]),
    "ffcu_dataset_device_column": (I, [VP, I, ctypes.POINTER(VP)]),
    "ffcu_nll_points": (I, [VP, VP, DP, I, DP, LLP, ULLP]),
    "ffcu_nll_points_partial": (I, [VP, VP, DP, I, DP, LLP, ULLP]),
    "ffcu_nll_points_device": (I, [VP, VP, DP, I, VP, VP, VP, ULLP]),
    "ffcu_nll_points_device_upload": (I, [VP, VP, DP, I, VP, VP, VP, VP, ULLP]),
    "ffcu_nll_grad": (I, [VP, VP, DP, I, DP, DP, LLP, ULLP]),
    "ffcu_grad_slot_count": (I, [VP, IP]),
    "ffcu_nll_grad_partial": (I, [VP, VP, DP, I, DP, LLP, ULLP]),
    "ffcu_nll_grad_finish": (I, [VP, DP, I, DP, D, DP, DP]),
    "ffcu_combine_pairs_device": (I, [VP, I, I, VP, VP]),
    "ffcu_extended_terms": (I, [VP, DP, I, D, DP]),
    "ffcu_probabilities_at": (I, [VP, VP, DP, DP]),
    "ffcu_eval_batch": (I, [VP, CP, VP, DP]),
    "ffcu_eval_batch_device": (I, [VP, CP, VP, VP, VP]),
    "ffcu_normalization": (I, [VP, CP, DP, DP]),
    "ffcu_model_set_device_normalization": (I, [VP, I]),
    "ffcu_model_device_normalization": (I, [VP]),
    "ffcu_device_normalization": (I, [VP, CP, DP, I, DP]),
    "ffcu_device_normalization_launches": (ULL, [VP]),
    "ffcu_plan_info": (I, [VP, IP, IP, IP]),
    "ffcu_plan_term": (I, [VP, I, IP, IP, IP, IP, IP]),
    "ffcu_point_constants": (I, [VP, DP, DP]),
    "ffcu_coef_derivatives": (I, [VP, DP, I, DP]),
    "ffcu_expr_eval": (I, [CP, ctypes.POINTER(CP), I, DP, I, DP]),
    "ffcu_expression_jit": (I, [I]),
    "ffcu_expression_jit_status": (CP, []),
    "ffcu_expression_jit_source": (I, [VP, I, CP, I]),
    "ffcu_last_launch_jit": (I, [VP]),
    "ffcu_last_launch_cached": (I, [VP]),
    "ffcu_plan_spec_source": (I, [VP, DP, I, I, ctypes.c_char_p, I]),
    "ffcu_plan_spec_min_work": (ctypes.c_double, [ctypes.c_double]),
    "ffcu_expression_jit_source_points": (I, [VP, DP, I, I, ctypes.c_char_p, I]),
    "ffcu_grad_spec_source": (I, [VP, I, CP, I]),
    "ffcu_last_grad_jit": (I, [VP]),
    "ffcu_soa_write": (I, [CP, ctypes.POINTER(CP), ctypes.POINTER(DP), I, LL]),
    "ffcu_dataset_save_soa": (I, [VP, CP]),
    "ffcu_dataset_load_soa": (I, [CP, ctypes.POINTER(VP), ctypes.POINTER(D)]),
    "ffcu_soa_info": (I, [CP, IP, ctypes.POINTER(LL)]),
    "ffcu_soa_column_name": (I, [CP, I, CP, I]),
    "ffcu_soa_read_host": (I, [CP, ctypes.POINTER(DP)]),
    "ffcu_model_pdf_count": (I, [VP]),
    "ffcu_model_pdf_name": (CP, [VP, I]),
    "ffcu_model_observable_count": (I, [VP]),
    "ffcu_model_observable_name": (CP, [VP, I]),
    "ffcu_fit_gradient": (I, [VP, VP, D, ctypes.c_long, ctypes.POINTER(VP)]),
    "ffcu_fit_gradient_opts": (I, [VP, VP, D, ctypes.c_long, I, ctypes.POINTER(VP)]),
    "ffcu_result_analytic_gradient": (I, [VP]),
    "ffcu_result_iterations": (I, [VP]),
    "ffcu_result_edm": (D, [VP]),
    "ffcu_result_launches": (ULL, [VP]),
    "ffcu_result_trace": (I, [VP, DP, I]),
    "ffcu_last_launch": (I, [VP, IP]),
    "ffcu_kernel_launches": (ULL, []),
    "ffcu_kernel_timer": (I, [I]),
    "ffcu_kernel_timer_read": (I, [DP, ULLP]),
    "ffcu_fp64_peak": (I, [DP, ctypes.POINTER(ctypes.c_float)]),
    "ffcu_fp64_issue_probe": (I, [I, DP]),
    "ffcu_math_probe": (I, [I, DP, DP, LL]),
    "ffcu_sample_host": (I, [VP, LL, ULL, ctypes.POINTER(DP), DP]),
    # event-sharded likelihood over several GPUs (csrc/shard.hpp)
    "ffcu_combine_shards_device": (I, [VP, I, I, I, VP, VP, VP, VP]),
    "ffcu_nccl_unique_id": (I, [VP]),
    "ffcu_nccl_version": (CP, []),
    "ffcu_shard_group_create_rank": (I, [VP, VP, LL, LL, VP, I, I, ctypes.POINTER(VP)]),
    "ffcu_shard_group_create_local": (I, [VP, ctypes.POINTER(CP), ctypes.POINTER(DP), I, LL, IP, I,
                                          ctypes.POINTER(VP)]),
    "ffcu_shard_group_free": (None, [VP]),
    "ffcu_shard_group_info": (I, [VP, IP, IP, LLP, LLP, LLP]),
    "ffcu_shard_group_nll_points": (I, [VP, DP, I, DP, LLP, ULLP]),
    "ffcu_shard_group_nll_points_device": (I, [VP, DP, I, VP, VP, VP, VP, ULLP]),
    "ffcu_shard_group_nll_grad": (I, [VP, DP, I, DP, DP, LLP, ULLP]),
    "ffcu_shard_group_fit": (I, [VP, D, ctypes.c_long, ctypes.POINTER(VP)]),
    "ffcu_shard_group_fit_gradient": (I, [VP, D, ctypes.c_long, I, ctypes.POINTER(VP)]),
}


def build(verbose=False):
    """Compile the CUDA/C++ sources into lib/libffit_b200.so (sm_100a)."""
    out = subprocess.run(["make", "-C", CSRC, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libffit_b200.so failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the GPU path has no fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
