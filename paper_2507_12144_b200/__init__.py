"""B200-native spherical-operator hot path of FourCastNet 3 (arXiv 2507.12144).

Drop-in for the operator API of the reference library spheretk (namespace ``sphere``):
SHT / inverse SHT, DISCO convolution, spectral convolution, the neural-operator block
epilogue and the lat/lon domain-decomposed distributed SHT + DISCO.  All compute runs
in libsphgpu.so (hand-written sm_100a CUDA behind the C ABI in include/sphere_gpu.h).
"""
from ._lib import LIB_PATH, SphError, SphInvalidArgument, launch_count  # noqa: F401
from .sphere import (  # noqa: F401
    EQUIANGULAR, GAUSSIAN, BlockWeights, DiscoOperator, FilterBasis, GridSpec, ShtPlan,
    SpectralCoeffs, SphericalField, assemble_disco, block_apply, block_epilogue,
    build_equiangular, build_gaussian, default_mmax, disco_apply, disco_transpose_apply, get_sht_plan,
    bilinear_resample, spectral_resample, ResamplePlan, DecoderPlan, decode_preclamp, angular_psd, spectral_crps_loss,
    isotropic_basis, morlet_basis, require_same_sampling, sht_forward, sht_inverse,
    sht_forward_adjoint, sht_inverse_adjoint,
    spectral_conv,
    spectral_mix,
)
