"""ctypes mirror of the C-ABI in include/rpd_b200.h.

The functions follow the reference C++ API of `namespace rpd`
(/root/reference/proj/include/rpd/*.hpp): same names, argument meaning,
buffer layouts and error behaviour.  Exceptions map the ABI status codes back
onto the reference's exception types:

  RPD_EINVAL       -> InvalidArgument   (std::invalid_argument, a ValueError)
  RPD_EDEGENERATE  -> DegenerateError   (std::runtime_error / DegenerateFitError)

`Context` binds one shared library.  The product library is the sm_100a CUDA
build (`paper_2012_10802_b200.load_library()`); the parity tests bind the same
class to the CPU oracle (oracle/_build/librpd_oracle.so) as the checker.
"""
from __future__ import annotations

import ctypes as C
import math
import dataclasses
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

RPD_OK, RPD_EINVAL, RPD_EDEGENERATE, RPD_ECUDA, RPD_ENOMEM, RPD_ECAPACITY = range(6)
STAGE_NAMES = ("sgm_bootstrap", "road_fit", "sgm_pt", "road_refit",
               "disparity_transform", "slic", "detect")  # pipeline.cpp:64-104
EIGHT_DIRECTIONS = ((1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, 1), (1, -1), (-1, -1))
INVALID = -1.0  # kInvalidDisparity, types.hpp:21


class RpdError(Exception):
    pass


class InvalidArgument(RpdError, ValueError):
    """std::invalid_argument."""


class DegenerateError(RpdError, RuntimeError):
    """std::runtime_error on degenerate data (DegenerateFitError in the pipeline)."""


class CudaError(RpdError, RuntimeError):
    pass


class CapacityError(RpdError):
    pass


class MissingSymbol(RpdError, NotImplementedError):
    """The bound library does not export this entry point."""


def _missing(path, name):
    def call(*_a, **_k):
        raise MissingSymbol(f"{path} does not export {name}")
    return call


# ------------------------------------------------------------------ structs --
class RoadModel(C.Structure):
    _fields_ = [("a0", C.c_double), ("a1", C.c_double), ("phi", C.c_double)]

    def __repr__(self):
        return f"RoadModel(a0={self.a0!r}, a1={self.a1!r}, phi={self.phi!r})"


class Config(C.Structure):
    _fields_ = [
        ("delta_pt", C.c_double), ("delta_dt", C.c_double), ("delta_pd", C.c_double),
        ("d_max", C.c_int32), ("d_max_pt", C.c_int32),
        ("lambda1", C.c_double), ("lambda2", C.c_double),
        ("census_window", C.c_int32), ("lr_threshold", C.c_double),
        ("superpixels", C.c_int32), ("compactness", C.c_double),
        ("slic_iterations", C.c_int32), ("hist_bin_width", C.c_double),
        ("tau_diag", C.c_double), ("border_margin", C.c_int32),
        ("min_superpixels", C.c_int32), ("connectivity", C.c_int32),
        ("roll_bracket", C.c_double), ("roll_tol", C.c_double),
        ("focal", C.c_double), ("baseline", C.c_double), ("cu", C.c_double),
        ("cv", C.c_double), ("sgm_paths", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}

    def copy(self):
        c = Config()
        C.pointer(c)[0] = self
        return c


class Center(C.Structure):
    _fields_ = [("cu", C.c_double), ("cv", C.c_double), ("value", C.c_double)]


class LineFit(C.Structure):
    _fields_ = [("model", RoadModel), ("e0min", C.c_double)]


class RoadFit(C.Structure):
    _fields_ = [("model", RoadModel), ("e0min", C.c_double), ("used", C.c_int64)]


class RectRoi(C.Structure):
    _fields_ = [("u0", C.c_int32), ("v0", C.c_int32), ("width", C.c_int32),
                ("height", C.c_int32)]


class Threshold(C.Structure):
    _fields_ = [("t_r", C.c_double), ("t_s", C.c_double), ("mu1", C.c_double),
                ("mu2", C.c_double), ("excluded_fraction", C.c_double),
                ("degenerate", C.c_int32)]


class Confusion(C.Structure):
    _fields_ = [("n_tp", C.c_int64), ("n_fp", C.c_int64), ("n_fn", C.c_int64),
                ("n_tn", C.c_int64)]

    def total(self) -> int:
        return self.n_tp + self.n_fp + self.n_fn + self.n_tn


class PixelReport(C.Structure):
    """PixelMetrics, evaluation.hpp:51-59."""
    _fields_ = [("counts", Confusion), ("precision", C.c_double), ("recall", C.c_double),
                ("accuracy", C.c_double), ("fscore", C.c_double),
                ("degenerate_precision", C.c_int32), ("degenerate_recall", C.c_int32)]


class InstanceReport(C.Structure):
    """InstanceReport, evaluation.hpp:91-95."""
    _fields_ = [("correct", C.c_int32), ("incorrect", C.c_int32), ("misdetection", C.c_int32)]


class StereoRig(C.Structure):
    """StereoRig, types.hpp:25-30."""
    _fields_ = [("focal", C.c_double), ("baseline", C.c_double), ("cu", C.c_double),
                ("cv", C.c_double)]


class Point3(C.Structure):
    _fields_ = [("x", C.c_float), ("y", C.c_float), ("z", C.c_float)]


class PotholeSpecC(C.Structure):
    """PotholeSpec, synth.hpp:12-18."""
    _fields_ = [("cu", C.c_double), ("cv", C.c_double), ("ru", C.c_double), ("rv", C.c_double),
                ("depth", C.c_double)]


class SceneSpecC(C.Structure):
    """SceneSpec, synth.hpp:20-30 (potholes as a pointer + count)."""
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("rig", StereoRig),
                ("a0", C.c_double), ("a1", C.c_double), ("phi_true", C.c_double),
                ("texture_seed", C.c_uint32), ("noise_sigma", C.c_double),
                ("n_potholes", C.c_int32), ("potholes", C.POINTER(PotholeSpecC))]


class BatchRangesC(C.Structure):
    """BatchRanges, synth.hpp:45-53."""
    _fields_ = [("depth_min", C.c_double), ("depth_max", C.c_double),
                ("radius_min", C.c_double), ("radius_max", C.c_double),
                ("a0_min", C.c_double), ("a0_max", C.c_double),
                ("a1_min", C.c_double), ("a1_max", C.c_double),
                ("phi_abs_max", C.c_double), ("noise_sigma", C.c_double),
                ("margin", C.c_int32)]


class DetectOut(C.Structure):
    _fields_ = [
        ("d0", C.POINTER(C.c_float)), ("d1", C.POINTER(C.c_float)),
        ("d2", C.POINTER(C.c_float)), ("d3", C.POINTER(C.c_float)),
        ("labels", C.POINTER(C.c_int32)), ("sp_labels", C.POINTER(C.c_int32)),
        ("centers", C.POINTER(Center)), ("centers_cap", C.c_int32),
        ("sp_count", C.c_int32), ("sp_spacing", C.c_double),
        ("coarse_fit", RoadFit), ("fit", RoadFit), ("threshold", Threshold),
        ("clamped", C.c_int64), ("n_potholes", C.c_int32),
        ("stage_ms", C.c_double * 7), ("total_ms", C.c_double),
    ]


@dataclass
class DetectResult:
    """DetectResult, pipeline.hpp:26-38."""
    d0: Optional[np.ndarray]
    d1: Optional[np.ndarray]
    d2: Optional[np.ndarray]
    d3: Optional[np.ndarray]
    labels: Optional[np.ndarray]
    sp_labels: Optional[np.ndarray]
    centers: Optional[np.ndarray]
    sp_count: int
    sp_spacing: float
    coarse_fit: RoadFit
    fit: RoadFit
    threshold: Threshold
    clamped: int
    n_potholes: int
    stage_ms: dict = field(default_factory=dict)
    total_ms: float = 0.0


@dataclass
class Histogram2D:
    """Histogram2D, segmentation.hpp:34-41."""
    bin_width: float
    origin: float
    counts: np.ndarray
    total: int

    def center(self, b):
        return self.origin + (b + 0.5) * self.bin_width


# ------------------------------------------------------------------ helpers --
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def slic_seed_count(h: int, w: int, p: int) -> int:
    """SLIC keeps at most its nu * nv seeds (segmentation.cpp:181-184)."""
    if h <= 0 or w <= 0 or p <= 0:
        return 1
    nu = max(1, int(math.floor(math.sqrt(p * w / h) + 0.5)))
    nv = max(1, int(math.floor(p / nu + 0.5)))
    return max(1, min(h * w, nu * nv))


def _on_device(a) -> bool:
    """A CUDA tensor (torch): the C-ABI takes device memory of the context's
    GPU wherever it takes a host buffer (abi_util.hpp: cudaMemcpyDefault)."""
    return getattr(a, "is_cuda", False) and hasattr(a, "data_ptr")


def _dev(a, dtype: str):
    if str(a.dtype) != "torch." + dtype or not a.is_contiguous():
        raise InvalidArgument(f"device arrays must be contiguous {dtype}")
    return a


def _ptr(a):
    if a is None:
        return None
    if _on_device(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return _dev(a, "float32") if _on_device(a) else np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return _dev(a, "float64") if _on_device(a) else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return _dev(a, "int32") if _on_device(a) else np.ascontiguousarray(a, dtype=np.int32)


def _fp(a):
    if a is not None and _on_device(a):
        return C.cast(a.data_ptr(), C.POINTER(C.c_float))
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    if a is not None and _on_device(a):
        return C.cast(a.data_ptr(), C.POINTER(C.c_int32))
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


_SIGS = {
    "rpd_abi_version": (C.c_int, []),
    "rpd_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "rpd_ctx_destroy": (None, [_vp]),
    "rpd_last_error": (C.c_char_p, [_vp]),
    "rpd_ctx_stream": (_vp, [_vp]),
    "rpd_config_default": (None, [C.POINTER(Config)]),
    "rpd_config_validate": (C.c_int, [_vp, C.POINTER(Config)]),
    "rpd_config_set": (C.c_int, [_vp, C.POINTER(Config), C.c_char_p, C.c_char_p]),
    "rpd_detect": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(Config),
                             C.POINTER(DetectOut)]),
    "rpd_detect_u8": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(Config),
                                C.POINTER(DetectOut)]),
    "rpd_compute_row_shifts": (C.c_int, [_vp, C.POINTER(RoadModel), C.c_int, C.c_int,
                                         C.c_double, _vp]),
    "rpd_warp_right_image": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp]),
    "rpd_restore_disparity": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp]),
    "rpd_census_cost_volume": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _vp, _vp]),
    "rpd_aggregate_costs": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int,
                                      C.c_float, C.c_float, _vp]),
    "rpd_swap_reference": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp]),
    "rpd_select_disparity": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp]),
    "rpd_consistency_filter": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_double]),
    "rpd_match_pair": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(RoadModel),
                                 C.POINTER(Config), C.c_int, _vp, _vp, _vp]),
    "rpd_sample_observations": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.POINTER(RectRoi),
                                          C.c_int64, _vp, _vp, _vp, C.POINTER(C.c_int64)]),
    "rpd_fit_line": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_double,
                               C.POINTER(LineFit)]),
    "rpd_estimate_roll": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_double, C.c_double,
                                    C.c_double, C.POINTER(RoadModel)]),
    "rpd_fit_road": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_double, C.c_double,
                               C.POINTER(RoadFit)]),
    "rpd_transform_disparity": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.POINTER(RoadModel),
                                          C.c_double, _vp, C.POINTER(C.c_int64)]),
    "rpd_slic": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _vp,
                           _vp, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    "rpd_pool_superpixels": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp]),
    "rpd_build_histogram": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double, _vp,
                                      C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64)]),
    "rpd_find_road_threshold": (C.c_int, [_vp, _vp, C.c_int64, C.c_double, C.c_double,
                                          C.c_int64, C.c_double, C.c_double,
                                          C.POINTER(Threshold)]),
    "rpd_connected_components": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp]),
    "rpd_detect_potholes": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(Threshold), C.c_int, C.c_int, C.c_int, _vp]),
    # evaluation.hpp
    "rpd_pep": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_double)]),
    "rpd_rmse": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "rpd_fscore": (C.c_double, [C.c_double, C.c_double]),
    "rpd_pixel_metrics": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(PixelReport)]),
    "rpd_instance_metrics": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_double,
                                       C.POINTER(InstanceReport)]),
    # road_geometry.hpp:64-73
    "rpd_rig_from_config": (StereoRig, [C.POINTER(Config), C.c_int, C.c_int]),
    "rpd_reproject": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.POINTER(StereoRig), _vp,
                                C.c_int64, C.POINTER(C.c_int64)]),
    "rpd_reproject_masked": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(StereoRig), _vp, C.c_int64,
                                       C.POINTER(C.c_int64)]),
    "rpd_reproject_instances": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(StereoRig), _vp, C.c_int64, _vp]),
    "rpd_closest_distance_error": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64,
                                             C.POINTER(C.c_double)]),
    # image_io.cpp per-pixel transforms
    "rpd_encode_disparity_u16": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_decode_disparity_u16": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_encode_labels_u16": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_encode_gray_u8": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_gray_from_rgb8": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_overlay_rgb8": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _vp]),
    "rpd_scene_spec_default": (None, [C.POINTER(SceneSpecC)]),
    "rpd_batch_ranges_default": (None, [C.POINTER(BatchRangesC)]),
    "rpd_scene_batch_spec": (C.c_int, [C.c_uint32, C.c_int32, C.POINTER(BatchRangesC),
                                       C.POINTER(SceneSpecC), C.POINTER(PotholeSpecC)]),
    "rpd_generate_scene": (C.c_int, [_vp, C.POINTER(SceneSpecC), _vp, _vp, _vp, _vp]),
}

class Stats(C.Structure):
    _fields_ = [("kernels_last_frame", C.c_int32), ("graph_replayed", C.c_int32),
                ("sgm_passes", C.c_int32), ("sgm_agg_ms", C.c_double * 2),
                ("sgm_agg_alg_bytes", C.c_double * 2), ("sgm_cells", C.c_double * 2),
                ("last_agg_kernel", C.c_int32), ("agg_segmented_ctas", C.c_int32),
                ("agg_segment_reruns", C.c_int64), ("slic_tiles_assigned", C.c_int64),
                ("slic_tiles_skipped", C.c_int64), ("slic_centres_moved", C.c_int64),
                ("slic_pixels_changed", C.c_int64)]


AGG_KERNELS = {0: "none", 1: "f32", 2: "u8_tma", 3: "u8"}  # RPD_AGG_*


class SgmDump(C.Structure):
    """rpd_sgm_dump (rpd_match_pair_dump_ex)."""
    _fields_ = [("cost", _vp), ("cost_right", _vp), ("agg_left", _vp), ("agg_right", _vp),
                ("disp_left", _vp), ("disp_right", _vp)]


_EXT_SIGS = {  # extensions of the product library (streaming, measurement)
    "rpd_input_buffers_u8": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp), C.POINTER(_vp)]),
    "rpd_detect_async_u8": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(Config)]),
    "rpd_detect_fetch": (C.c_int, [_vp, C.POINTER(DetectOut)]),
    "rpd_detect_async": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(Config)]),
    "rpd_generate_scenes_device": (C.c_int, [_vp, C.c_int, C.POINTER(SceneSpecC), _vp, _vp, _vp,
                                             _vp]),
    "rpd_detect_async_host_u8": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(Config)]),
    "rpd_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "rpd_host_free": (None, [_vp]),
    "rpd_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "rpd_ctx_stats": (C.c_int, [_vp, C.POINTER(Stats)]),
    "rpd_debug_sincos": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
    "rpd_debug_scan": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "rpd_debug_guard_check": (C.c_int, [_vp, C.POINTER(C.c_longlong), C.c_char_p, C.c_int]),
    "rpd_debug_guard_selftest": (C.c_int, [_vp, C.c_size_t]),
}
_SIGS["rpd_match_pair_dump"] = (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(RoadModel),
                                          C.POINTER(Config), C.c_int, _vp, _vp, _vp, _vp, _vp])

_SIGS["rpd_match_pair_dump_ex"] = (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int,
                                             C.POINTER(RoadModel), C.POINTER(Config), C.c_int,
                                             C.POINTER(SgmDump)])

ABI_SYMBOLS = tuple(_SIGS)
EXTENSION_SYMBOLS = tuple(_EXT_SIGS)


class Library:
    """One loaded shared library exporting the rpd_* C-ABI."""

    def __init__(self, path: str):
        self.path = str(path)
        self.dll = C.CDLL(self.path)
        # The product and the restated oracle export every symbol; the literal
        # reference wrapper (oracle/_ref) only the hot-path subset — calls to
        # a missing one raise MissingSymbol.
        self.missing = set()
        for name, (res, args) in _SIGS.items():
            if not hasattr(self.dll, name):
                self.missing.add(name)
                setattr(self.dll, name, _missing(self.path, name))
                continue
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args
        self.has_streaming = all(hasattr(self.dll, n) for n in _EXT_SIGS)
        if self.has_streaming:
            for name, (res, args) in _EXT_SIGS.items():
                fn = getattr(self.dll, name)
                fn.restype = res
                fn.argtypes = args
        if self.dll.rpd_abi_version() != 1:
            raise RpdError(f"{path}: unexpected ABI version")

    def pinned_empty(self, shape, dtype):
        """numpy array over page-locked host memory (rpd_host_alloc); freed
        when the array is garbage collected."""
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        p = _vp()
        if self.dll.rpd_host_alloc(nbytes, C.byref(p)) != RPD_OK:
            raise MemoryError("rpd_host_alloc failed")
        buf = (C.c_uint8 * max(nbytes, 1)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)
        import weakref
        weakref.finalize(buf, self.dll.rpd_host_free, p.value)
        return arr

    def default_config(self, **overrides) -> Config:
        cfg = Config()
        self.dll.rpd_config_default(C.byref(cfg))
        for k, v in overrides.items():
            if not hasattr(cfg, k):
                raise InvalidArgument(f"config: unknown key '{k}'")
            setattr(cfg, k, v)
        return cfg

    def context(self, device: int = 0, max_h: int = 0, max_w: int = 0, max_levels: int = 0):
        return Context(self, device, max_h, max_w, max_levels)


class Context:
    """rpd_ctx: per (host thread, device) state.  Methods mirror namespace rpd."""

    def __init__(self, lib: Library, device=0, max_h=0, max_w=0, max_levels=0):
        self.lib = lib
        self.dll = lib.dll
        h = _vp()
        self._check(self.dll.rpd_ctx_create(device, max_h, max_w, max_levels, C.byref(h)),
                    ctx=None)
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self.dll.rpd_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self):
        return self.dll.rpd_ctx_stream(self.handle)

    def _check(self, st, ctx="self"):
        if st == RPD_OK:
            return
        msg = ""
        if ctx is not None and getattr(self, "handle", None):
            raw = self.dll.rpd_last_error(self.handle)
            msg = raw.decode() if raw else ""
        exc = {RPD_EINVAL: InvalidArgument, RPD_EDEGENERATE: DegenerateError,
               RPD_ECUDA: CudaError, RPD_ECAPACITY: CapacityError}.get(st, RpdError)
        raise exc(msg or f"rpd status {st}")

    # -------------------------------------------------------------- config --
    def validate(self, cfg: Config):
        self._check(self.dll.rpd_config_validate(self.handle, C.byref(cfg)))

    def config_set(self, cfg: Config, key: str, value):
        self._check(self.dll.rpd_config_set(self.handle, C.byref(cfg), key.encode(),
                                            str(value).encode()))

    # ------------------------------------------------------------ pipeline --
    def detect(self, left, right, cfg: Config, want=("d0", "d1", "d2", "d3", "labels",
                                                      "sp_labels", "centers")) -> DetectResult:
        """detect_potholes_pipeline (pipeline.hpp:43-44).  uint8 inputs use the
        exact uint8 entry point, anything else is passed as float32."""
        u8 = isinstance(left, np.ndarray) and left.dtype == np.uint8
        if u8:
            left = np.ascontiguousarray(left)
            right = np.ascontiguousarray(right)
        else:
            left = _f32(left)
            right = _f32(right)
        if left.shape != right.shape or left.ndim != 2:
            raise InvalidArgument("match_pair: dimension mismatch")
        h, w = left.shape
        bufs = {k: (np.empty((h, w), np.float32) if k in want else None)
                for k in ("d0", "d1", "d2", "d3")}
        bufs["labels"] = np.empty((h, w), np.int32) if "labels" in want else None
        bufs["sp_labels"] = np.empty((h, w), np.int32) if "sp_labels" in want else None
        cap = slic_seed_count(h, w, cfg.superpixels) if "centers" in want else 0
        centers = (Center * max(cap, 1))() if cap else None
        out = DetectOut()
        for k in ("d0", "d1", "d2", "d3"):
            setattr(out, k, _fp(bufs[k]))
        out.labels = _ip(bufs["labels"])
        out.sp_labels = _ip(bufs["sp_labels"])
        out.centers = C.cast(centers, C.POINTER(Center)) if centers is not None else None
        out.centers_cap = cap
        fn = self.dll.rpd_detect_u8 if u8 else self.dll.rpd_detect
        self._check(fn(self.handle, _ptr(left), _ptr(right), h, w, C.byref(cfg), C.byref(out)))
        cent = None
        if centers is not None:
            cent = np.array([(c.cu, c.cv, c.value) for c in centers[:min(out.sp_count, cap)]],
                            dtype=np.float64).reshape(-1, 3)
        return DetectResult(
            d0=bufs["d0"], d1=bufs["d1"], d2=bufs["d2"], d3=bufs["d3"],
            labels=bufs["labels"], sp_labels=bufs["sp_labels"], centers=cent,
            sp_count=out.sp_count, sp_spacing=out.sp_spacing, coarse_fit=out.coarse_fit,
            fit=out.fit, threshold=out.threshold, clamped=out.clamped,
            n_potholes=out.n_potholes,
            stage_ms={n: out.stage_ms[i] for i, n in enumerate(STAGE_NAMES)},
            total_ms=out.total_ms)

    # ------------------------------------------- streaming / measurement --
    def input_buffers_u8(self, h: int, w: int):
        """Device pointers (ints) of the context's uint8 input buffers."""
        l, r = _vp(), _vp()
        self._check(self.dll.rpd_input_buffers_u8(self.handle, h, w, C.byref(l), C.byref(r)))
        return l.value, r.value

    def detect_async_u8(self, d_left: int, d_right: int, h: int, w: int, cfg: Config):
        self._check(self.dll.rpd_detect_async_u8(self.handle, d_left, d_right, h, w,
                                                 C.byref(cfg)))

    def detect_async_host_u8(self, left_ptr: int, right_ptr: int, h: int, w: int, cfg: Config):
        """Enqueue H2D (async from pinned memory) + the frame; fetch() completes it."""
        self._check(self.dll.rpd_detect_async_host_u8(self.handle, left_ptr, right_ptr, h, w,
                                                      C.byref(cfg)))

    def detect_async(self, d_left: int, d_right: int, h: int, w: int, cfg: Config):
        """Device-resident float32 images (e.g. from generate_scenes_device)."""
        self._check(self.dll.rpd_detect_async(self.handle, d_left, d_right, h, w, C.byref(cfg)))

    def fetch(self, out: Optional[DetectOut] = None) -> DetectOut:
        out = out if out is not None else DetectOut()
        self._check(self.dll.rpd_detect_fetch(self.handle, C.byref(out)))
        return out

    def debug_sincos(self, x):
        x = _f64(x)
        s = np.empty_like(x)
        c = np.empty_like(x)
        self._check(self.dll.rpd_debug_sincos(self.handle, _ptr(x), x.shape[0], _ptr(s), _ptr(c)))
        return s, c

    def debug_scan(self, flags):
        """(exclusive prefix sums, total) of int32 flags on the device (scan.cuh)."""
        a = np.ascontiguousarray(flags, dtype=np.int32)
        out = np.empty_like(a)
        tot = C.c_int32(0)
        self._check(self.dll.rpd_debug_scan(self.handle, _ptr(a), a.shape[0], _ptr(out),
                                            C.byref(tot)))
        return out, tot.value

    def guard_check(self):
        """(corrupted guard bytes, first buffer) — checked build only (-1 otherwise)."""
        n = C.c_longlong(0)
        buf = C.create_string_buffer(128)
        self._check(self.dll.rpd_debug_guard_check(self.handle, C.byref(n), buf, 128))
        return n.value, buf.value.decode()

    def set_profiling(self, enable: bool):
        self._check(self.dll.rpd_ctx_set_profiling(self.handle, 1 if enable else 0))

    def stats(self) -> Stats:
        s = Stats()
        self._check(self.dll.rpd_ctx_stats(self.handle, C.byref(s)))
        return s

    def detect_raw(self, left_ptr: int, right_ptr: int, h: int, w: int, cfg: Config,
                   out: DetectOut, u8: bool = True):
        """rpd_detect(_u8) on raw host pointers (e.g. pinned buffers)."""
        fn = self.dll.rpd_detect_u8 if u8 else self.dll.rpd_detect
        self._check(fn(self.handle, left_ptr, right_ptr, h, w, C.byref(cfg), C.byref(out)))
        return out

    # --------------------------------------------------------- perspective --
    def compute_row_shifts(self, model: RoadModel, width: int, height: int, delta_pt: float):
        out = np.empty(height, np.float64)
        self._check(self.dll.rpd_compute_row_shifts(self.handle, C.byref(model), width, height,
                                                    delta_pt, _ptr(out)))
        return out

    def warp_right_image(self, right, shifts):
        right = _f32(right)
        shifts = _f64(shifts)
        h, w = right.shape
        if shifts.shape[0] != h:
            raise InvalidArgument("warp_right_image: table length != image height")
        img = np.empty((h, w), np.float32)
        iv = np.empty((h, w), np.uint8)
        self._check(self.dll.rpd_warp_right_image(self.handle, _ptr(right), h, w, _ptr(shifts),
                                                  _ptr(img), _ptr(iv)))
        return img, iv

    def restore_disparity(self, d0, shifts):
        d0 = _f32(d0)
        shifts = _f64(shifts)
        h, w = d0.shape
        if shifts.shape[0] != h:
            raise InvalidArgument("restore_disparity: table length != map height")
        d1 = np.empty((h, w), np.float32)
        self._check(self.dll.rpd_restore_disparity(self.handle, _ptr(d0), h, w, _ptr(shifts),
                                                   _ptr(d1)))
        return d1

    # ----------------------------------------------------------------- SGM --
    def census_cost_volume(self, left, right_warped, d_max: int, window: int, in_view=None):
        left = _f32(left)
        right_warped = _f32(right_warped)
        if left.shape != right_warped.shape:
            raise InvalidArgument("census_cost_volume: dimension mismatch")
        h, w = left.shape
        iv = None if in_view is None else np.ascontiguousarray(in_view, dtype=np.uint8)
        out = np.empty((h, w, max(d_max, 0) + 1), np.float32)
        self._check(self.dll.rpd_census_cost_volume(self.handle, _ptr(left), _ptr(right_warped),
                                                    h, w, d_max, window, _ptr(iv), _ptr(out)))
        return out

    def aggregate_costs(self, costs, lambda1=8.0, lambda2=32.0,
                        directions: Sequence = EIGHT_DIRECTIONS):
        costs = _f32(costs)
        h, w, n = costs.shape
        dirs = np.ascontiguousarray(np.array(directions, dtype=np.int32).reshape(-1, 2))
        out = np.empty_like(costs)
        self._check(self.dll.rpd_aggregate_costs(self.handle, _ptr(costs), h, w, n - 1,
                                                 _ptr(dirs), dirs.shape[0], lambda1, lambda2,
                                                 _ptr(out)))
        return out

    def swap_reference(self, costs):
        costs = _f32(costs)
        h, w, n = costs.shape
        out = np.empty_like(costs)
        self._check(self.dll.rpd_swap_reference(self.handle, _ptr(costs), h, w, n - 1,
                                                _ptr(out)))
        return out

    def select_disparity(self, aggregated):
        agg = _f32(aggregated)
        h, w, n = agg.shape
        out = np.empty((h, w), np.float32)
        self._check(self.dll.rpd_select_disparity(self.handle, _ptr(agg), h, w, n - 1,
                                                  _ptr(out)))
        return out

    def consistency_filter(self, left_disp, right_disp, threshold: float):
        """Returns the filtered copy (the reference mutates in place)."""
        left = _f32(left_disp).copy()
        right = _f32(right_disp)
        h, w = left.shape
        self._check(self.dll.rpd_consistency_filter(self.handle, _ptr(left), _ptr(right), h, w,
                                                    threshold))
        return left

    def match_pair(self, left, right, model: RoadModel, cfg: Config, d_max: int):
        left = _f32(left)
        right = _f32(right)
        if left.shape != right.shape:
            raise InvalidArgument("match_pair: dimension mismatch")
        h, w = left.shape
        d0 = np.empty((h, w), np.float32)
        d1 = np.empty((h, w), np.float32)
        sh = np.empty(h, np.float64)
        self._check(self.dll.rpd_match_pair(self.handle, _ptr(left), _ptr(right), h, w,
                                            C.byref(model), C.byref(cfg), d_max, _ptr(d0),
                                            _ptr(d1), _ptr(sh)))
        return d0, d1, sh

    def match_pair_dump(self, left, right, model: RoadModel, cfg: Config, d_max: int):
        """Intermediates of match_pair: (cost, agg_left, agg_right, disp_left, disp_right)."""
        left = _f32(left)
        right = _f32(right)
        h, w = left.shape
        vols = [np.empty((h, w, d_max + 1), np.float32) for _ in range(3)]
        maps = [np.empty((h, w), np.float32) for _ in range(2)]
        self._check(self.dll.rpd_match_pair_dump(self.handle, _ptr(left), _ptr(right), h, w,
                                                 C.byref(model), C.byref(cfg), d_max,
                                                 *[_ptr(v) for v in vols],
                                                 *[_ptr(m) for m in maps]))
        return (*vols, *maps)

    def match_pair_dump_ex(self, left, right, model: RoadModel, cfg: Config, d_max: int):
        """match_pair intermediates incl. the right-reference costs, as a dict:
        cost, cost_right, agg_left, agg_right (H x W x L), disp_left, disp_right."""
        left = _f32(left)
        right = _f32(right)
        h, w = left.shape
        res = {k: np.empty((h, w, d_max + 1), np.float32)
               for k in ("cost", "cost_right", "agg_left", "agg_right")}
        res.update({k: np.empty((h, w), np.float32) for k in ("disp_left", "disp_right")})
        d = SgmDump(**{k: v.ctypes.data for k, v in res.items()})
        self._check(self.dll.rpd_match_pair_dump_ex(self.handle, _ptr(left), _ptr(right), h, w,
                                                    C.byref(model), C.byref(cfg), d_max,
                                                    C.byref(d)))
        return res

    # ------------------------------------------------------- road geometry --
    def sample_observations(self, d1, roi: Optional[RectRoi] = None, cap: int = 100000):
        d1 = _f32(d1)
        h, w = d1.shape
        n = min(h * w, cap)
        d = np.empty(max(n, 1), np.float64)
        u = np.empty_like(d)
        v = np.empty_like(d)
        k = C.c_int64(0)
        self._check(self.dll.rpd_sample_observations(
            self.handle, _ptr(d1), h, w, C.byref(roi) if roi is not None else None, cap,
            _ptr(d), _ptr(u), _ptr(v), C.byref(k)))
        k = k.value
        return d[:k].copy(), u[:k].copy(), v[:k].copy()

    def fit_line(self, d, u, v, phi: float) -> LineFit:
        d, u, v = _f64(d), _f64(u), _f64(v)
        out = LineFit()
        self._check(self.dll.rpd_fit_line(self.handle, _ptr(d), _ptr(u), _ptr(v), d.shape[0],
                                          phi, C.byref(out)))
        return out

    def estimate_roll(self, d, u, v, lo: float, hi: float, tol: float) -> RoadModel:
        d, u, v = _f64(d), _f64(u), _f64(v)
        out = RoadModel()
        self._check(self.dll.rpd_estimate_roll(self.handle, _ptr(d), _ptr(u), _ptr(v),
                                               d.shape[0], lo, hi, tol, C.byref(out)))
        return out

    def fit_road(self, d, u, v, bracket: float, tol: float) -> RoadFit:
        d, u, v = _f64(d), _f64(u), _f64(v)
        out = RoadFit()
        self._check(self.dll.rpd_fit_road(self.handle, _ptr(d), _ptr(u), _ptr(v), d.shape[0],
                                          bracket, tol, C.byref(out)))
        return out

    def transform_disparity(self, d1, model: RoadModel, delta_dt: float):
        d1 = _f32(d1)
        h, w = d1.shape
        d2 = np.empty_like(d1)
        clamped = C.c_int64(0)
        self._check(self.dll.rpd_transform_disparity(self.handle, _ptr(d1), h, w,
                                                     C.byref(model), delta_dt, _ptr(d2),
                                                     C.byref(clamped)))
        return d2, clamped.value

    # -------------------------------------------------------- segmentation --
    def slic(self, d2, p: int, compactness: float, iterations: int):
        d2 = _f32(d2)
        h, w = d2.shape
        labels = np.empty((h, w), np.int32)
        cap = slic_seed_count(h, w, p)
        centers = (Center * cap)()
        count = C.c_int32(0)
        spacing = C.c_double(0)
        self._check(self.dll.rpd_slic(self.handle, _ptr(d2), h, w, p, compactness, iterations,
                                      _ptr(labels), centers, cap, C.byref(count),
                                      C.byref(spacing)))
        cent = np.array([(c.cu, c.cv, c.value) for c in centers[:min(count.value, cap)]],
                        dtype=np.float64).reshape(-1, 3)
        return labels, cent, count.value, spacing.value

    def pool_superpixels(self, d2, sp_labels, sp_count: int):
        d2 = _f32(d2)
        lab = _i32(sp_labels)
        h, w = d2.shape
        if lab.shape != d2.shape:
            raise InvalidArgument("pool_superpixels: dimension mismatch")
        d3 = np.empty_like(d2)
        self._check(self.dll.rpd_pool_superpixels(self.handle, _ptr(d2), _ptr(lab), sp_count,
                                                  h, w, _ptr(d3)))
        return d3

    def build_histogram(self, d2, bin_width: float) -> Histogram2D:
        d2 = _f32(d2)
        h, w = d2.shape
        n = C.c_int64(0)
        origin = C.c_double(0)
        total = C.c_int64(0)
        st = self.dll.rpd_build_histogram(self.handle, _ptr(d2), h, w, bin_width, None, 0,
                                          C.byref(n), C.byref(origin), C.byref(total))
        if st not in (RPD_OK, RPD_ECAPACITY):
            self._check(st)
        nn = n.value
        counts = np.zeros((nn, nn), np.int64)
        if nn > 0:
            self._check(self.dll.rpd_build_histogram(self.handle, _ptr(d2), h, w, bin_width,
                                                     _ptr(counts), nn, C.byref(n),
                                                     C.byref(origin), C.byref(total)))
        return Histogram2D(bin_width, origin.value, counts, total.value)

    def find_road_threshold(self, hist: Histogram2D, delta_pd: float, tau: float = 3.0):
        counts = np.ascontiguousarray(hist.counts, dtype=np.int64)
        n = counts.shape[0] if counts.ndim == 2 else 0
        out = Threshold()
        self._check(self.dll.rpd_find_road_threshold(self.handle, _ptr(counts), n,
                                                     hist.bin_width, hist.origin, hist.total,
                                                     delta_pd, tau, C.byref(out)))
        return out

    def connected_components(self, mask, connectivity: int = 8):
        mask = _i32(mask)
        h, w = mask.shape
        out = np.empty_like(mask)
        self._check(self.dll.rpd_connected_components(self.handle, _ptr(mask), h, w,
                                                      connectivity, _ptr(out)))
        return out

    def detect_potholes(self, d3, sp_labels, sp_spacing: float, thr: Threshold,
                        border_margin: int, min_superpixels: int, connectivity: int = 8):
        d3 = _f32(d3)
        lab = _i32(sp_labels)
        h, w = d3.shape
        out = np.empty((h, w), np.int32)
        self._check(self.dll.rpd_detect_potholes(self.handle, _ptr(d3), _ptr(lab), sp_spacing,
                                                 h, w, C.byref(thr), border_margin,
                                                 min_superpixels, connectivity, _ptr(out)))
        return out


    # ---- evaluation.hpp:14-149 ---------------------------------------------
    def _pair(self, a, b, conv):
        a, b = conv(a), conv(b)
        if a.shape != b.shape:
            raise InvalidArgument("evaluation: dimension mismatch")
        return a, b

    def pep(self, est, gt, eps: float) -> float:
        est, gt = self._pair(est, gt, _f32)
        out = C.c_double()
        self._check(self.dll.rpd_pep(self.handle, _ptr(est), _ptr(gt), est.shape[0],
                                     est.shape[1], eps, C.byref(out)))
        return out.value

    def rmse(self, est, gt) -> float:
        est, gt = self._pair(est, gt, _f32)
        out = C.c_double()
        self._check(self.dll.rpd_rmse(self.handle, _ptr(est), _ptr(gt), est.shape[0],
                                      est.shape[1], C.byref(out)))
        return out.value

    def fscore(self, precision: float, recall: float) -> float:
        return self.dll.rpd_fscore(precision, recall)

    def pixel_metrics(self, pred, gt_mask) -> PixelReport:
        pred, gt_mask = self._pair(pred, gt_mask, _i32)
        out = PixelReport()
        self._check(self.dll.rpd_pixel_metrics(self.handle, _ptr(pred), _ptr(gt_mask),
                                               pred.shape[0], pred.shape[1], C.byref(out)))
        return out

    def instance_metrics(self, pred, gt_instances, iou_min: float = 0.5) -> InstanceReport:
        pred, gt_instances = self._pair(pred, gt_instances, _i32)
        out = InstanceReport()
        self._check(self.dll.rpd_instance_metrics(self.handle, _ptr(pred), _ptr(gt_instances),
                                                  pred.shape[0], pred.shape[1], iou_min,
                                                  C.byref(out)))
        return out


    # ---- road_geometry.hpp:64-73 -------------------------------------------
    def rig_from_config(self, cfg: Config, width: int, height: int) -> StereoRig:
        return self.dll.rpd_rig_from_config(C.byref(cfg), width, height)

    def reproject(self, d1, rig: StereoRig, labels=None, label: int = 0) -> np.ndarray:
        """PointCloud as an (n, 3) float32 array (reproject / reproject_masked)."""
        d1 = _f32(d1)
        h, w = d1.shape
        cap = h * w
        out = np.empty((max(cap, 1), 3), np.float32)
        n = C.c_int64()
        if labels is None:
            st = self.dll.rpd_reproject(self.handle, _ptr(d1), h, w, C.byref(rig), _ptr(out), cap,
                                        C.byref(n))
        else:
            lab = _i32(labels)
            if lab.shape != d1.shape:
                raise InvalidArgument("reproject_masked: dimension mismatch")
            st = self.dll.rpd_reproject_masked(self.handle, _ptr(d1), _ptr(lab), h, w, label,
                                               C.byref(rig), _ptr(out), cap, C.byref(n))
        self._check(st)
        return out[:n.value].copy()

    def reproject_instances(self, d1, labels, max_label: int, rig: StereoRig):
        """[cloud of label 1, ..., cloud of label max_label]."""
        d1, lab = _f32(d1), _i32(labels)
        h, w = d1.shape
        cap = h * w
        out = np.empty((max(cap, 1), 3), np.float32)
        off = np.zeros(max_label + 1, np.int64)
        self._check(self.dll.rpd_reproject_instances(self.handle, _ptr(d1), _ptr(lab), h, w,
                                                     max_label, C.byref(rig), _ptr(out), cap,
                                                     _ptr(off)))
        return [out[off[k - 1]:off[k]].copy() for k in range(1, max_label + 1)]

    def closest_distance_error(self, test, truth) -> float:
        t = np.ascontiguousarray(np.asarray(test, np.float32).reshape(-1, 3))
        g = np.ascontiguousarray(np.asarray(truth, np.float32).reshape(-1, 3))
        out = C.c_double()
        self._check(self.dll.rpd_closest_distance_error(self.handle, _ptr(t), t.shape[0], _ptr(g),
                                                        g.shape[0], C.byref(out)))
        return out.value


    # ---- image_io.cpp per-pixel transforms ---------------------------------
    def encode_disparity_u16(self, d) -> np.ndarray:
        d = _f32(d)
        out = np.empty(d.shape, np.uint16)
        self._check(self.dll.rpd_encode_disparity_u16(self.handle, _ptr(d), *d.shape, _ptr(out)))
        return out

    def decode_disparity_u16(self, s) -> np.ndarray:
        s = np.ascontiguousarray(s, np.uint16)
        out = np.empty(s.shape, np.float32)
        self._check(self.dll.rpd_decode_disparity_u16(self.handle, _ptr(s), *s.shape, _ptr(out)))
        return out

    def encode_labels_u16(self, labels) -> np.ndarray:
        lab = _i32(labels)
        out = np.empty(lab.shape, np.uint16)
        self._check(self.dll.rpd_encode_labels_u16(self.handle, _ptr(lab), *lab.shape, _ptr(out)))
        return out

    def encode_gray_u8(self, img) -> np.ndarray:
        img = _f32(img)
        out = np.empty(img.shape, np.uint8)
        self._check(self.dll.rpd_encode_gray_u8(self.handle, _ptr(img), *img.shape, _ptr(out)))
        return out

    def gray_from_rgb8(self, rgb) -> np.ndarray:
        rgb = np.ascontiguousarray(rgb, np.uint8)
        h, w = rgb.shape[:2]
        out = np.empty((h, w), np.float32)
        self._check(self.dll.rpd_gray_from_rgb8(self.handle, _ptr(rgb), h, w, _ptr(out)))
        return out

    def overlay_rgb8(self, img, labels) -> np.ndarray:
        img, lab = _f32(img), _i32(labels)
        if img.shape != lab.shape:
            raise DegenerateError("overlay: dimension mismatch")
        out = np.empty(img.shape + (3,), np.uint8)
        self._check(self.dll.rpd_overlay_rgb8(self.handle, _ptr(img), _ptr(lab), *img.shape,
                                              _ptr(out)))
        return out

    # ------------------------------------------- synth.hpp (§8(f) row 4) --
    def generate_scene(self, spec):
        """generate_scene (synth.cpp:94-149) -> (left, right, gt_disparity, gt_mask).
        `spec` is a scenes.SceneSpec (or anything with its attributes)."""
        cs, keep = scene_spec_c(spec)
        h, w = cs.height, cs.width
        left = np.empty((h, w), np.float32)
        right = np.empty((h, w), np.float32)
        gt = np.empty((h, w), np.float32)
        mask = np.empty((h, w), np.int32)
        self._check(self.dll.rpd_generate_scene(self.handle, C.byref(cs), _ptr(left), _ptr(right),
                                                _ptr(gt), _ptr(mask)))
        del keep
        return left, right, gt, mask

    def generate_scenes_device(self, specs, d_left: int, d_right: int, d_gt: int, d_mask: int):
        """Streaming extension: len(specs) same-size scenes into device buffers."""
        arr = (SceneSpecC * len(specs))()
        keep = []
        for i, sp in enumerate(specs):
            arr[i], k = scene_spec_c(sp)
            keep.append(k)
        self._check(self.dll.rpd_generate_scenes_device(self.handle, len(specs), arr, d_left,
                                                        d_right, d_gt, d_mask))


def scene_spec_c(spec):
    """ctypes SceneSpecC of a SceneSpec-like object; returns (struct, keepalive)."""
    pots = list(getattr(spec, "potholes", []) or [])
    parr = (PotholeSpecC * max(len(pots), 1))()
    for i, p in enumerate(pots):
        parr[i] = PotholeSpecC(p.cu, p.cv, p.ru, p.rv, p.depth)
    rig = getattr(spec, "rig", None)
    rig_c = StereoRig(rig.focal, rig.baseline, rig.cu, rig.cv) if rig is not None else \
        StereoRig(700.0, 0.12, 0.0, 0.0)
    cs = SceneSpecC(int(spec.width), int(spec.height), rig_c, float(spec.a0), float(spec.a1),
                    float(spec.phi_true), int(spec.texture_seed) & 0xFFFFFFFF,
                    float(spec.noise_sigma), len(pots), parr)
    return cs, parr


def model(a0=0.0, a1=0.0, phi=0.0) -> RoadModel:
    return RoadModel(a0, a1, phi)


def threshold(t_r=0.0, t_s=0.0, mu1=0.0, mu2=0.0, excluded_fraction=0.0, degenerate=0):
    return Threshold(t_r, t_s, mu1, mu2, excluded_fraction, degenerate)
