"""B200-native extended correlation / convolution (arXiv 2006.13188 hot path).

The reference's operator API (xcorr_fast, xconv_fast, smooth_adaptive, ...)
backed by hand-written sm_100a CUDA kernels behind the C ABI of
include/xconv_b200.h.  See DESIGN.md.
"""
from .engine import (DetectionResult, FreqFilter2, Peak, Response2, SmoothResult, VoteFilter,
                     XConvPlan, XformField, XformKind, XMode, anglemax, build_optimal_filter,
                     build_vote_filter, decompose_rotation2, decompose_scale2, detect_pattern,
                     fft2, find_peaks, inner_dc_value, reconstruct, render_component,
                     smooth_adaptive, xconv_fast, xcorr_fast)
from .lic import anisotropic_gaussian, lic, white_noise
from .contour import ContourMatch, ContourScene, match_contours, rasterize_contours
from .engine3d import (Response3, SphFilter3, decompose_rotation3, reconstruct3, steer_filter3,
                       render_sph_component, rotation3d, sph_harm, wigner_d, xconv_fast_3d,
                       xcorr_fast_3d)

__all__ = ["DetectionResult", "FreqFilter2", "Peak", "Response2", "SmoothResult", "VoteFilter",
           "XConvPlan", "XformField", "XformKind", "XMode", "anglemax", "build_optimal_filter",
           "build_vote_filter", "decompose_rotation2", "decompose_scale2", "detect_pattern",
           "fft2", "find_peaks", "inner_dc_value", "reconstruct", "render_component",
           "smooth_adaptive", "xconv_fast", "xcorr_fast", "Response3", "SphFilter3",
           "decompose_rotation3", "reconstruct3", "render_sph_component", "rotation3d",
           "sph_harm", "wigner_d", "xconv_fast_3d", "xcorr_fast_3d", "anisotropic_gaussian", "lic",
           "white_noise", "ContourMatch", "ContourScene", "match_contours", "rasterize_contours",
           "steer_filter3"]
