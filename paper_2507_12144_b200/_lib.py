"""ctypes binding of libsphgpu.so (the C ABI in include/sphere_gpu.h).

The shared library is the product: it is built in-tree for sm_100a
(``python -m paper_2507_12144_b200.build``).  Importing this module without the
library raises immediately -- there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPH_LIBSPHGPU: load another build of the library (same-box A/B runs, profiles/lib_ab.sh)
LIB_PATH = os.environ.get("SPH_LIBSPHGPU") or os.path.join(_HERE, "libsphgpu.so")

SPH_OK = 0
SPH_ERR_INVALID_ARGUMENT = 1
SPH_ERR_RUNTIME = 2
SPH_ERR_CUDA = 3
SPH_ERR_NCCL = 4
SPH_ERR_OOM = 5

SPH_EQUIANGULAR = 0
SPH_GAUSSIAN = 1
SPH_PREC_3XTF32 = 0
SPH_PREC_TF32 = 1
SPH_PREC_FP32_SIMT = 2
SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD = 0x10
SPH_FLAG_ADJOINT = 0x20
SPH_LAYOUT_DENSE_LM = 0
SPH_LAYOUT_INTERNAL = 1
SPH_BASIS_MORLET = 0
SPH_BASIS_ISOTROPIC = 1

# every symbol declared in include/sphere_gpu.h (checked by tests/test_capi.py)
EXPORTS = [
    "sph_last_error", "sph_version", "sph_launch_count", "sph_profile_enable",
    "sph_profile_read", "sph_grid",
    "sph_sht_plan_create", "sph_sht_plan_destroy", "sph_sht_coeffs_elems",
    "sph_sht_workspace_bytes", "sph_sht_forward", "sph_sht_inverse", "sph_sht_roundtrip_host",
    "sph_sht_fft_stage", "sph_sht_legendre_stage", "sph_sht_stage_workspace_bytes",
    "sph_disco_plan_create", "sph_disco_plan_destroy", "sph_disco_plan_info",
    "sph_disco_workspace_bytes", "sph_disco_apply", "sph_disco_input_rows",
    "sph_disco_rows_workspace_bytes", "sph_disco_apply_rows", "sph_disco_transpose_workspace_bytes",
    "sph_disco_transpose_apply", "sph_resample_plan_create", "sph_resample_plan_destroy",
    "sph_resample_workspace_bytes", "sph_bilinear_resample", "sph_decoder_plan_create",
    "sph_decoder_plan_destroy", "sph_decoder_workspace_bytes", "sph_decoder_apply", "sph_psd_from_coeffs",
    "sph_spectral_crps_from_coeffs", "sph_weighted_crps",
    "sph_spectral_conv", "sph_spectral_conv_workspace_bytes", "sph_spectral_mix", "sph_block_epilogue",
    "sph_comm_id_bytes", "sph_comm_unique_id", "sph_comm_create", "sph_comm_destroy", "sph_comm_coords",
    "sph_comm_traffic_csv", "sph_comm_traffic_reset", "sph_dist_sht_plan_create", "sph_dist_sht_plan_destroy",
    "sph_dist_sht_local", "sph_dist_sht_workspace_bytes", "sph_dist_sht_forward", "sph_dist_sht_inverse",
    "sph_dist_disco_plan_create", "sph_dist_disco_plan_destroy", "sph_dist_disco_local",
    "sph_dist_disco_workspace_bytes", "sph_dist_disco_apply", "sph_dist_sht_describe", "sph_dist_disco_describe",
]


class SphError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class SphInvalidArgument(SphError, ValueError):
    """std::invalid_argument of the reference."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2507_12144_b200/build.py` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_double)
    L.sph_last_error.restype = C.c_char_p
    L.sph_version.restype = C.c_char_p
    L.sph_launch_count.restype = C.c_uint64
    L.sph_profile_enable.argtypes = [i32]
    L.sph_profile_read.argtypes = [C.c_char_p, C.c_size_t]
    L.sph_grid.argtypes = [i32, i64, i64, dp, dp]
    L.sph_sht_plan_create.argtypes = [i32, i64, i64, i64, i64, i32, C.POINTER(vp)]
    L.sph_sht_plan_destroy.argtypes = [vp]
    L.sph_sht_coeffs_elems.argtypes = [vp, i64, i32]
    L.sph_sht_coeffs_elems.restype = i64
    L.sph_sht_workspace_bytes.argtypes = [vp, i64]
    L.sph_sht_workspace_bytes.restype = i64
    L.sph_sht_forward.argtypes = [vp, vp, i64, vp, i32, vp, vp]
    L.sph_sht_inverse.argtypes = [vp, vp, i64, i32, vp, vp, vp]
    L.sph_sht_roundtrip_host.argtypes = [vp, vp, i64, vp, i64]
    L.sph_sht_fft_stage.argtypes = [vp, vp, i64, i64, vp, vp]
    L.sph_sht_legendre_stage.argtypes = [vp, vp, i64, i64, i64, vp, vp, vp]
    L.sph_sht_stage_workspace_bytes.argtypes = [vp, i64, i64]
    L.sph_sht_stage_workspace_bytes.restype = i64
    L.sph_disco_plan_create.argtypes = [i32, i64, i64, i32, i64, i64, i32, C.c_double, i32,
                                        C.POINTER(vp)]
    L.sph_disco_plan_destroy.argtypes = [vp]
    L.sph_disco_plan_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    L.sph_disco_workspace_bytes.argtypes = [vp, i64, i64, i64]
    L.sph_disco_workspace_bytes.restype = i64
    L.sph_disco_apply.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, vp]
    L.sph_disco_input_rows.argtypes = [vp, i64, i64, C.POINTER(i64), C.POINTER(i64)]
    L.sph_disco_rows_workspace_bytes.argtypes = [vp, i64, i64, i64, i64, i64]
    L.sph_disco_rows_workspace_bytes.restype = i64
    L.sph_disco_apply_rows.argtypes = [vp, vp, i64, i64, i64, i64, vp, i64, i64, i64, vp, vp, vp]
    L.sph_disco_transpose_workspace_bytes.argtypes = [vp, i64, i64, i64]
    L.sph_disco_transpose_workspace_bytes.restype = i64
    L.sph_disco_transpose_apply.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, vp]
    L.sph_resample_plan_create.argtypes = [vp, i64, i64, vp, i64, i64, C.POINTER(vp)]
    L.sph_resample_plan_destroy.argtypes = [vp]
    L.sph_resample_workspace_bytes.argtypes = [vp, i64]
    L.sph_resample_workspace_bytes.restype = i64
    L.sph_bilinear_resample.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sph_decoder_plan_create.argtypes = [vp, vp, i64, i64, C.POINTER(vp)]
    L.sph_decoder_plan_destroy.argtypes = [vp]
    L.sph_decoder_workspace_bytes.argtypes = [vp, i64, i64, i64]
    L.sph_decoder_workspace_bytes.restype = i64
    L.sph_decoder_apply.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, vp]
    L.sph_psd_from_coeffs.argtypes = [vp, i64, i64, i64, vp, vp]
    L.sph_spectral_crps_from_coeffs.argtypes = [vp, vp, i64, i64, i64, i64, i64, C.c_int, vp, vp]
    L.sph_weighted_crps.argtypes = [vp, vp, vp, i64, i64, i64, C.c_int, vp, vp]
    L.sph_spectral_conv.argtypes = [vp, vp, vp, i64, i64, i64, i64, vp, vp, vp]
    L.sph_spectral_mix.argtypes = [vp, vp, vp, i64, i64, i64, i64, vp, vp, vp]
    L.sph_spectral_conv_workspace_bytes.argtypes = [vp, i64, i64, i64]
    L.sph_spectral_conv_workspace_bytes.restype = i64
    L.sph_block_epilogue.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp]
    ip = C.POINTER(i64)
    L.sph_comm_id_bytes.restype = i64
    L.sph_comm_unique_id.argtypes = [vp]
    L.sph_comm_create.argtypes = [vp, i64, i64, ip, C.POINTER(vp)]
    L.sph_comm_destroy.argtypes = [vp]
    L.sph_comm_coords.argtypes = [vp, ip]
    L.sph_comm_traffic_csv.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.sph_comm_traffic_reset.argtypes = [vp]
    L.sph_dist_sht_plan_create.argtypes = [vp, vp, i64, C.POINTER(vp)]
    L.sph_dist_sht_plan_destroy.argtypes = [vp]
    L.sph_dist_sht_local.argtypes = [vp, ip]
    L.sph_dist_sht_workspace_bytes.argtypes = [vp]
    L.sph_dist_sht_workspace_bytes.restype = i64
    L.sph_dist_sht_forward.argtypes = [vp, vp, vp, vp, vp]
    L.sph_dist_sht_inverse.argtypes = [vp, vp, vp, vp, vp]
    L.sph_dist_disco_plan_create.argtypes = [vp, vp, i64, i64, C.POINTER(vp)]
    L.sph_dist_disco_plan_destroy.argtypes = [vp]
    L.sph_dist_disco_local.argtypes = [vp, ip]
    L.sph_dist_disco_workspace_bytes.argtypes = [vp]
    L.sph_dist_disco_workspace_bytes.restype = i64
    L.sph_dist_disco_apply.argtypes = [vp, vp, vp, vp, vp, vp]
    L.sph_dist_sht_describe.argtypes = [i64] * 8 + [C.c_int, ip, i64, ip]
    L.sph_dist_disco_describe.argtypes = [i64] * 9 + [ip, ip, C.c_int, ip, i64, ip]
    for name in EXPORTS:
        getattr(L, name)  # AttributeError if a declared symbol is not exported
    return L


lib = _load()


def check(rc: int) -> None:
    if rc != SPH_OK:
        msg = lib.sph_last_error().decode()
        if rc == SPH_ERR_INVALID_ARGUMENT:
            raise SphInvalidArgument(rc, msg)
        raise SphError(rc, msg)


def launch_count() -> int:
    return int(lib.sph_launch_count())


def profile_enable(on: bool = True) -> None:
    lib.sph_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel name: (launches, total_ms, work)} since the previous read."""
    buf = C.create_string_buffer(1 << 16)
    check(lib.sph_profile_read(buf, 1 << 16))
    out = {}
    for line in buf.value.decode().splitlines()[1:]:
        n, c, t, w = line.split(",")
        out[n] = (int(c), float(t), float(w))
    return out
