"""ctypes binding of liblgs.so (include/lgs.h).

This is the Python side of the C ABI: plain structs and pointers, no torch types.  It fails
loudly when the library is missing -- there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblgs.so")

LGS_OK, LGS_EINVAL, LGS_ECUDA, LGS_ENOMEM, LGS_ENODEV, LGS_EIO = range(6)
LGS_MEM_HOST, LGS_MEM_DEVICE, LGS_MEM_HOST_MAPPED = 0, 1, 2
LGS_OPT_FULL_TILE_LISTS, LGS_OPT_RADIX_DEPTH_ORDER, LGS_OPT_FUSED_EAGER, LGS_OPT_HOST_GRAD_DELTA = 0, 1, 2, 3
LGS_OPT_SPECULATIVE_PLANS = 4

_fp = C.POINTER(C.c_float)


class LgsRenderConfig(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "near_plane", "dilation", "alpha_clamp", "alpha_skip", "transmittance_min", "radius_sigma")]


class LgsCamera(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("t", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class LgsGaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("feature_dim", C.c_int32), ("sh_degree", C.c_int32),
                ("positions", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("opacity_logits", C.c_void_p), ("sh", C.c_void_p), ("features", C.c_void_p),
                ("memory", C.c_int32)]


class LgsImages(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("feat", C.c_void_p), ("acc", C.c_void_p),
                ("memory", C.c_int32)]


class LgsMapGrads(C.Structure):
    _fields_ = [("position", C.c_void_p), ("rotation", C.c_void_p), ("log_scale", C.c_void_p),
                ("opacity_logit", C.c_void_p), ("sh", C.c_void_p), ("feature", C.c_void_p),
                ("memory", C.c_int32), ("accumulate", C.c_int32)]


class LgsL1Targets(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("feat", C.c_void_p), ("memory", C.c_int32)]


class LgsCotangents(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("feat", C.c_void_p), ("memory", C.c_int32),
                ("rgb_shape", C.c_int32 * 3), ("depth_shape", C.c_int32 * 3), ("feat_shape", C.c_int32 * 3)]


class LgsPruneConfig(C.Structure):
    _fields_ = [("k_neighbors", C.c_int32), ("tau_dist", C.c_double), ("tau_sim", C.c_double),
                ("alpha_min", C.c_double), ("scale_max", C.c_double)]


class LgsRenderStats(C.Structure):
    _fields_ = [("visible", C.c_int64), ("pairs", C.c_int64), ("tiles", C.c_int64), ("max_tile_list", C.c_int64),
                ("listed", C.c_int64), ("active", C.c_int64), ("host_rows", C.c_int64)]


class LgsDecoder(C.Structure):
    _fields_ = [("high_dim", C.c_int32), ("hidden", C.c_int32), ("low_dim", C.c_int32), ("w1", C.c_void_p),
                ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p), ("memory", C.c_int32)]


class LgsKeyframe(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("feat_gt", C.c_void_p), ("memory", C.c_int32)]


class LgsLossWeights(C.Structure):
    _fields_ = [("w_l1", C.c_double), ("w_depth", C.c_double), ("w_feat", C.c_double)]


class LgsLossBreakdown(C.Structure):
    _fields_ = [("l_rgb", C.c_double), ("l_depth", C.c_double), ("l_feat", C.c_double), ("l_total", C.c_double),
                ("ssim", C.c_double), ("depth_pixels", C.c_int64)]


class LgsAdamConfig(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lr_position", "lr_rotation", "lr_log_scale", "lr_opacity", "lr_color",
                                          "lr_sh_rest", "lr_feature", "beta1", "beta2", "eps")]


class LgsCommId(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 128)]


# (name, restype, argtypes) for every symbol declared in include/lgs.h
SIGNATURES = [
    ("lgs_version", C.c_char_p, []),
    ("lgs_last_error", C.c_char_p, []),
    ("lgs_render_config_default", LgsRenderConfig, []),
    ("lgs_ctx_create", C.c_int, [C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("lgs_ctx_set_full_tile_lists", C.c_int, [C.c_void_p, C.c_int32]),
    ("lgs_ctx_set_option", C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    ("lgs_ctx_transfer_bytes", C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("lgs_ctx_destroy", C.c_int, [C.c_void_p]),
    ("lgs_ctx_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("lgs_ctx_synchronize", C.c_int, [C.c_void_p]),
    ("lgs_ctx_launch_count", C.c_int64, [C.c_void_p]),
    ("lgs_ctx_layer_div", C.c_int32, [C.c_void_p]),
    ("lgs_map_create", C.c_int, [C.c_void_p, C.POINTER(LgsGaussians), C.POINTER(C.c_void_p)]),
    ("lgs_map_update", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsGaussians)]),
    ("lgs_map_destroy", C.c_int, [C.c_void_p]),
    ("lgs_map_size", C.c_int64, [C.c_void_p]),
    ("lgs_render_forward", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsCamera), C.POINTER(LgsRenderConfig),
                                     C.POINTER(LgsL1Targets), C.POINTER(LgsImages), C.POINTER(C.c_void_p)]),
    ("lgs_render", C.c_int, [C.c_void_p, C.POINTER(LgsGaussians), C.POINTER(LgsCamera), C.POINTER(LgsRenderConfig),
                             C.POINTER(LgsImages), C.POINTER(C.c_void_p)]),
    ("lgs_render_backward", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsCotangents), C.POINTER(LgsMapGrads), _fp]),
    ("lgs_render_backward_l1", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads), _fp]),
    ("lgs_saved_l1_loss", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
    ("lgs_saved_stats", C.c_int, [C.c_void_p, C.POINTER(LgsRenderStats)]),
    ("lgs_saved_destroy", C.c_int, [C.c_void_p]),
    ("lgs_debug_projected", C.c_int, [C.c_void_p, C.c_void_p] + [C.c_void_p] * 9),
    ("lgs_debug_tile_keys", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("lgs_debug_pixel_state", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("lgs_grads_flat_size", C.c_int64, [C.c_int64, C.c_int32, C.c_int32]),
    ("lgs_phase_name", C.c_char_p, [C.c_int32]),
    ("lgs_ctx_profile", C.c_int, [C.c_void_p, C.c_int32]),
    ("lgs_ctx_phase_times", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]),
    ("lgs_saved_work", C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("lgs_loss_weights_default", LgsLossWeights, []),
    ("lgs_mapping_loss", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsImages), C.POINTER(LgsKeyframe),
                                   C.POINTER(LgsDecoder), C.POINTER(LgsLossWeights), C.POINTER(LgsLossBreakdown)]),
    ("lgs_render_backward_loss", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads), _fp]),
    ("lgs_render_backward_loss_async", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads), C.c_void_p]),
    ("lgs_debug_cotangents", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("lgs_coverage_mask", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_int64)]),
    ("lgs_adam_config_default", LgsAdamConfig, []),
    ("lgs_adam_create", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsAdamConfig), C.POINTER(C.c_void_p)]),
    ("lgs_adam_destroy", C.c_int, [C.c_void_p]),
    ("lgs_adam_steps", C.c_int64, [C.c_void_p]),
    ("lgs_adam_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads)]),
    ("lgs_map_download", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsGaussians)]),
    ("lgs_map_file_info", C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    ("lgs_map_file_read", C.c_int, [C.c_char_p, C.c_int32, C.POINTER(LgsGaussians), C.c_void_p]),
    ("lgs_map_file_write", C.c_int, [C.c_char_p, C.POINTER(LgsGaussians), C.c_void_p]),
    ("lgs_map_load", C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("lgs_map_save", C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_void_p]),
    ("lgs_prune_config_default", LgsPruneConfig, []),
    ("lgs_find_language_redundant", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsPruneConfig), C.c_void_p,
                                              C.c_int32, C.POINTER(C.c_int64)]),
    ("lgs_find_geometric", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsPruneConfig), C.c_void_p, C.c_int32,
                                     C.POINTER(C.c_int64)]),
    ("lgs_prune", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(LgsPruneConfig), C.c_void_p, C.c_void_p,
                            C.c_int32, C.POINTER(C.c_int64)]),
    ("lgs_prune_stats", C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("lgs_plan_create", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsCamera), C.POINTER(LgsRenderConfig),
                                  C.POINTER(LgsL1Targets), C.POINTER(LgsImages), C.POINTER(LgsMapGrads), C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
    ("lgs_plan_run", C.c_int, [C.c_void_p, C.c_void_p]),
    ("lgs_plan_sync", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    ("lgs_plan_set_camera", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsCamera)]),
    ("lgs_plan_elapsed_ms", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("lgs_plan_set_profiling", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    ("lgs_plan_phase_times", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("lgs_plan_launches", C.c_int64, [C.c_void_p]),
    ("lgs_plan_recaptures", C.c_int64, [C.c_void_p]),
    ("lgs_plan_speculative", C.c_int32, [C.c_void_p]),
    ("lgs_plan_destroy", C.c_int, [C.c_void_p]),
    ("lgs_comm_unique_id", C.c_int, [C.POINTER(LgsCommId)]),
    ("lgs_comm_init", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(LgsCommId)]),
    ("lgs_comm_destroy", C.c_int, [C.c_void_p]),
    ("lgs_allreduce_grads", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads)]),
    ("lgs_allreduce_f32", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    ("lgs_allreduce_grads_sparse", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    ("lgs_comm_set_timeout", C.c_int, [C.c_void_p, C.c_int64]),
    ("lgs_debug_sparse_reduce_simulated", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.POINTER(LgsMapGrads)),
                                                   C.c_int32, C.c_int64, C.POINTER(C.c_int64),
                                                   C.POINTER(C.c_int32)]),
    ("lgs_allreduce_grads_sparse_async", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads)]),
    ("lgs_allreduce_grads_sparse_wait", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(LgsMapGrads),
                                                 C.POINTER(C.c_int64)]),
]

LGS_PHASE_COUNT = 13

_lib = None


class LgsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"lgs status {status}: {msg}")
        self.status = status


class LgsInvalidArgument(LgsError, ValueError):
    """LGS_EINVAL -- the reference's std::invalid_argument (renderer.cpp:176-178)."""


class LgsIoError(LgsError, OSError):
    """LGS_EIO -- the reference's lego::IoError (errors.hpp:21) for map files."""


def load(path: str | None = None):
    """Load liblgs.so (raises if it is missing: the CUDA path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"{p} is missing: build it with __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(p)
    for name, res, args in SIGNATURES:
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status):
    if status != LGS_OK:
        msg = load().lgs_last_error().decode(errors="replace")
        if status == LGS_EINVAL:
            raise LgsInvalidArgument(status, msg)
        if status == LGS_EIO:
            raise LgsIoError(status, msg)
        raise LgsError(status, msg)
