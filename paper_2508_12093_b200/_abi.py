"""ctypes binding of include/hestat_gpu.h (libhestat_gpu.so, built in-tree).

Loading fails loudly when the shared library is missing: there is no CPU
fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhestat_gpu.so")


class hs_params(C.Structure):
    _fields_ = [("slot_count", C.c_uint64), ("max_level", C.c_int32), ("scale_bits", C.c_int32),
                ("quantize", C.c_int32), ("auto_bootstrap", C.c_int32), ("debug_checks", C.c_int32),
                ("_pad", C.c_int32)]


class hs_meter(C.Structure):
    _fields_ = [("mul_ct", C.c_uint64), ("mul_pt", C.c_uint64), ("add", C.c_uint64),
                ("rotate", C.c_uint64), ("bootstrap", C.c_uint64)]


class hs_invroot_cfg(C.Structure):
    _fields_ = [("n", C.c_int32), ("cheb_degree", C.c_int32), ("newton_iters", C.c_int32),
                ("baseline_mode", C.c_int32), ("baseline_iters", C.c_int32), ("_pad", C.c_int32)]


class hs_sign_cfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("folds", C.c_int32), ("polys", C.POINTER(C.c_double)),
                ("poly_len", C.POINTER(C.c_uint64)), ("npolys", C.c_uint64)]


CT = C.c_void_p
CTX = C.c_void_p
PCT = C.POINTER(C.c_void_p)
DP = C.POINTER(C.c_double)


class hs_column(C.Structure):
    _fields_ = [("chunks", PCT), ("n_chunks", C.c_uint64), ("n_valid", C.c_uint64)]


TARGET_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)

_SIGS = {
    "hs_last_error": (C.c_char_p, []),
    "hs_version": (C.c_char_p, []),
    "hs_init": (C.c_int, [C.c_int]),
    "hs_sync": (C.c_int, []),
    "hs_stream": (C.c_void_p, []),
    "hs_set_fused": (C.c_int, [C.c_int]),
    "hs_kernel_launches": (C.c_uint64, []),
    "hs_diag_fp64_rate": (C.c_int, [C.c_int, DP]),
    "hs_graph_begin": (C.c_int, []),
    "hs_graph_end": (C.c_int, [C.POINTER(C.c_void_p)]),
    "hs_graph_launch": (C.c_int, [C.c_void_p]),
    "hs_graph_destroy": (None, [C.c_void_p]),
    "hs_params_validate": (C.c_int, [C.POINTER(hs_params)]),
    "hs_ctx_create": (C.c_int, [C.POINTER(hs_params), C.c_uint64, C.POINTER(CTX)]),
    "hs_ctx_clone": (C.c_int, [CTX, C.POINTER(CTX)]),
    "hs_ctx_destroy": (None, [CTX]),
    "hs_ctx_params": (C.c_int, [CTX, C.POINTER(hs_params)]),
    "hs_ctx_meter": (C.c_int, [CTX, C.POINTER(hs_meter)]),
    "hs_ctx_set_meter": (C.c_int, [CTX, C.POINTER(hs_meter)]),
    "hs_ctx_rng_seed": (C.c_uint64, [CTX]),
    "hs_ct_new": (C.c_int, [DP, C.c_uint64, C.c_int32, PCT]),
    "hs_ct_retain": (CT, [CT]),
    "hs_ct_release": (None, [CT]),
    "hs_ct_level": (C.c_int32, [CT]),
    "hs_ct_size": (C.c_uint64, [CT]),
    "hs_ct_read": (C.c_int, [CT, DP, C.c_uint64]),
    "hs_encrypt": (C.c_int, [CTX, DP, C.c_uint64, PCT]),
    "hs_decrypt": (C.c_int, [CTX, CT, C.c_uint64, DP]),
    "hs_add_ct": (C.c_int, [CTX, CT, CT, PCT]),
    "hs_sub_ct": (C.c_int, [CTX, CT, CT, PCT]),
    "hs_add_pt": (C.c_int, [CTX, CT, C.c_double, PCT]),
    "hs_mul_ct": (C.c_int, [CTX, CT, CT, PCT]),
    "hs_mul_pt": (C.c_int, [CTX, CT, C.c_double, PCT]),
    "hs_mul_pt_vec": (C.c_int, [CTX, CT, DP, C.c_uint64, PCT]),
    "hs_rotate": (C.c_int, [CTX, CT, C.c_int64, PCT]),
    "hs_bootstrap": (C.c_int, [CTX, CT, PCT]),
    "hs_sum_all_slots": (C.c_int, [CTX, CT, C.c_uint64, PCT]),
    "hs_add_ct_batch": (C.c_int, [CTX, PCT, PCT, C.c_uint64, PCT]),
    "hs_sub_ct_batch": (C.c_int, [CTX, PCT, PCT, C.c_uint64, PCT]),
    "hs_mul_ct_batch": (C.c_int, [CTX, PCT, PCT, C.c_uint64, PCT]),
    "hs_add_pt_batch": (C.c_int, [CTX, PCT, C.c_double, C.c_uint64, PCT]),
    "hs_mul_pt_batch": (C.c_int, [CTX, PCT, C.c_double, C.c_uint64, PCT]),
    "hs_rotate_batch": (C.c_int, [CTX, PCT, C.c_int64, C.c_uint64, PCT]),
    "hs_scaled_target": (C.c_double, [C.c_int, C.c_double, C.c_double]),
    "hs_cheb_eval_depth": (C.c_int32, [C.c_int32]),
    "hs_fit": (C.c_int, [TARGET_FN, C.c_void_p, C.c_int32, C.c_double, C.c_double, DP]),
    "hs_fit_target": (C.c_int, [C.c_int, C.c_double, C.c_int32, C.c_double, C.c_double, DP]),
    "hs_eval_plain": (C.c_double, [DP, C.c_uint64, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int32)]),
    "hs_eval_encrypted": (C.c_int, [CTX, DP, C.c_uint64, C.c_double, C.c_double, CT, PCT]),
    "hs_newton_loop": (C.c_int, [CTX, CT, CT, C.c_int32, C.c_int32, C.c_uint64, PCT]),
    "hs_newton_refine": (C.c_int, [CTX, CT, CT, C.c_int32, C.c_int32, C.c_uint64, PCT]),
    "hs_crypto_invsqrt": (C.c_int, [CTX, CT, C.c_double, C.POINTER(hs_invroot_cfg), C.c_uint64, PCT]),
    "hs_baseline_invsqrt": (C.c_int, [CTX, CT, C.c_double, C.c_int32, C.c_uint64, PCT]),
    "hs_crypto_inv": (C.c_int, [CTX, CT, C.c_double, C.POINTER(hs_invroot_cfg), C.c_uint64, PCT]),
    "hs_crypto_sqrt": (C.c_int, [CTX, CT, C.c_double, C.c_int32, C.c_uint64, PCT]),
    "hs_crypto_sign": (C.c_int, [CTX, CT, C.POINTER(hs_sign_cfg), PCT]),
    "hs_encode_column": (C.c_int, [CTX, DP, C.c_uint64, PCT, C.POINTER(C.c_uint64)]),
    "hs_decode_column": (C.c_int, [CTX, C.POINTER(hs_column), DP]),
    "hs_encode_column_async": (C.c_int, [CTX, DP, C.c_uint64, PCT, C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)]),
    "hs_decode_column_async": (C.c_int, [CTX, C.POINTER(hs_column), DP, C.POINTER(C.c_void_p)]),
    "hs_pending_wait": (C.c_int, [C.c_void_p]),
    "hs_pending_release": (None, [C.c_void_p]),
    "hs_mean_scaled": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, PCT]),
    "hs_variance_to_scale": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, PCT]),
    "hs_variance_scaled": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, PCT]),
    "hs_moments": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, PCT, PCT]),
    "hs_znorm": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, C.POINTER(hs_invroot_cfg), PCT]),
    "hs_kurtosis": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, C.POINTER(hs_invroot_cfg), PCT]),
    "hs_skewness": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, C.POINTER(hs_invroot_cfg), PCT]),
    "hs_coeff_variation": (C.c_int, [CTX, C.POINTER(hs_column), C.c_double, C.POINTER(hs_sign_cfg),
                                     C.POINTER(hs_invroot_cfg), PCT]),
    "hs_pearson": (C.c_int, [CTX, C.POINTER(hs_column), C.POINTER(hs_column), C.c_double,
                             C.POINTER(hs_invroot_cfg), PCT]),
    "hs_pearson_table": (C.c_int, [CTX, C.POINTER(C.POINTER(hs_column)), C.c_uint32, C.c_double,
                                   C.POINTER(hs_invroot_cfg), PCT]),
    "hs_znorm_batch": (C.c_int, [CTX, C.POINTER(C.POINTER(hs_column)), C.c_uint32, C.c_double,
                                 C.POINTER(hs_invroot_cfg), PCT]),
    "hs_synthetic_uniform": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_double, DP]),
    "hs_synthetic_grid": (C.c_int, [C.c_uint64, C.c_double, C.c_double, DP]),
    "hs_two_subrange_grid": (C.c_int, [C.c_uint64, C.c_double, C.c_double, DP]),
    "hs_mre": (C.c_int, [DP, DP, C.c_uint64, DP]),
    "hs_relative_error": (C.c_int, [C.c_double, C.c_double, DP]),
    "hs_plain": (C.c_int, [C.c_int, DP, C.c_uint64, DP, DP]),
}



class hs_rns_spec(C.Structure):  # include/hestat_rns.h
    _fields_ = [("logN", C.c_uint32), ("L", C.c_uint32), ("K", C.c_uint32), ("dnum", C.c_uint32),
                ("logq0", C.c_uint32), ("logq", C.c_uint32), ("logp", C.c_uint32), ("h", C.c_uint32),
                ("seed", C.c_uint64)]


U64P = C.POINTER(C.c_uint64)
RNS = C.c_void_p
_SIGS.update({
    "hs_rns_create": (C.c_int, [C.POINTER(hs_rns_spec), C.POINTER(C.c_void_p)]),
    "hs_rns_destroy": (C.c_int, [RNS]),
    "hs_rns_primes": (C.c_int, [RNS, U64P, C.c_uint32]),
    "hs_rns_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "hs_rns_free": (C.c_int, [C.c_void_p]),
    "hs_rns_upload": (C.c_int, [C.c_void_p, U64P, C.c_uint64]),
    "hs_rns_download": (C.c_int, [U64P, C.c_void_p, C.c_uint64]),
    "hs_rns_prepare_relin": (C.c_int, [RNS]),
    "hs_rns_prepare_rotation": (C.c_int, [RNS, C.c_int64]),
    "hs_rns_secret": (C.c_int, [RNS, C.c_void_p]),
    "hs_rns_random_ct": (C.c_int, [RNS, C.c_uint32, C.c_uint64, C.c_void_p]),
    "hs_rns_encode": (C.c_int, [C.c_uint32, DP, C.c_uint64, C.c_double, C.POINTER(C.c_int64)]),
    "hs_rns_decode": (C.c_int, [C.c_uint32, C.POINTER(C.c_int64), C.c_double, DP, C.c_uint64]),
    "hs_rns_encode_gpu": (C.c_int, [C.c_uint32, DP, C.c_uint64, C.c_double, DP]),
    "hs_rns_decode_gpu": (C.c_int, [C.c_uint32, DP, C.c_double, DP, C.c_uint64]),
    "hs_rns_add": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_rns_sub": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_rns_add_const": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint32]),
    "hs_rns_mul_const": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint32]),
    "hs_rns_encrypt_coeffs": (C.c_int, [RNS, C.c_uint32, C.POINTER(C.c_int64), C.c_uint64, C.c_void_p]),
    "hs_rns_encrypt": (C.c_int, [RNS, C.c_uint32, DP, C.c_uint64, C.c_double, C.c_uint64, C.c_void_p]),
    "hs_rns_decrypt_coeffs": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.POINTER(C.c_int64)]),
    "hs_rns_decrypt": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_double, DP, C.c_uint64]),
    "hs_rns_eval_create": (C.c_int, [RNS, C.POINTER(hs_params), C.POINTER(C.c_void_p)]),
    "hs_rns_eval_destroy": (C.c_int, [C.c_void_p]),
    "hs_rns_eval_meter": (C.c_int, [C.c_void_p, C.POINTER(hs_meter)]),
    "hs_rns_eval_set_meter": (C.c_int, [C.c_void_p, C.POINTER(hs_meter)]),
    "hs_rns_eval_stat": (C.c_int, [C.c_void_p, C.c_int, DP, C.c_uint64, DP, C.c_uint64, C.c_double,
                                   C.POINTER(hs_invroot_cfg), DP, C.c_uint64, C.POINTER(C.c_int32)]),
    "hs_rns_ntt": (C.c_int, [RNS, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]),
    "hs_rns_mul_relin": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_rns_mul_relin_rescale": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_rns_rescale": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_rns_rescale_mul_const": (C.c_int, [RNS, C.c_uint32, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint32]),
    "hs_rns_rotate": (C.c_int, [RNS, C.c_uint32, C.c_int64, C.c_void_p, C.c_void_p, C.c_uint32]),
    "hs_ctx_create_rns": (C.c_int, [C.POINTER(hs_params), C.c_uint64, C.POINTER(hs_rns_spec), C.c_int,
                                    C.POINTER(CTX)]),
    "hs_ctx_backend": (C.c_int, [CTX]),
    "hs_ctx_rns_spec": (C.c_int, [CTX, C.POINTER(hs_rns_spec), C.POINTER(C.c_int)]),
    "hs_ct_backend": (C.c_int, [CT]),
})

_lib = None


def lib():
    """The loaded libhestat_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(no CPU fallback exists for the product path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def symbols():
    """Every exported entry point declared in include/hestat_gpu.h and include/hestat_rns.h."""
    return sorted(_SIGS)
