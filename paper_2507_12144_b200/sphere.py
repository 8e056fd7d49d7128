"""Python mirror of the reference operator API (namespace ``sphere`` of spheretk).

Same names, argument meaning and error behaviour as the reference
(/root/reference/proj/include/sphere/*.hpp), computed by libsphgpu.so on the GPU:

=====================================  ==============================================
reference                              here
=====================================  ==============================================
build_equiangular / build_gaussian     same (grid.hpp:69 / :91), fp64 host arrays
SphericalField [C][nlat][nlon]         ``SphericalField`` (data: fp32 CUDA tensor,
                                       leading batch dims allowed: [..., C, nlat, nlon])
SpectralCoeffs [C][lmax][mmax]         ``SpectralCoeffs`` (complex64 CUDA tensor)
sht_forward (harmonics.hpp:126-169)    ``sht_forward`` -- Gaussian only, like the ref
sht_inverse (harmonics.hpp:173-205)    ``sht_inverse``
morlet_basis / isotropic_basis         same (convolution.hpp:73-81)
assemble_disco (convolution.hpp:141)   ``assemble_disco`` -> DiscoOperator (device plan)
disco_apply (convolution.hpp:181)      ``disco_apply``
spectral_conv (convolution.hpp:286)    ``spectral_conv``
block_apply (model.hpp:337)            ``block_apply``
=====================================  ==============================================

``std::invalid_argument`` surfaces as ``ValueError`` (``SphInvalidArgument``), other
failures as ``RuntimeError``.  Tensors are torch CUDA tensors: torch is used for
device memory and streams only; every operator runs in the library's own kernels.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field as dc_field
from typing import Dict, Optional

import numpy as np
import torch

from . import _lib as L
from ._lib import check

PI = math.pi
EQUIANGULAR = L.SPH_EQUIANGULAR
GAUSSIAN = L.SPH_GAUSSIAN
PRECISIONS = {"3xtf32": L.SPH_PREC_3XTF32, "tf32": L.SPH_PREC_TF32, "fp32": L.SPH_PREC_FP32_SIMT}


# ------------------------------------------------------------------- grids
@dataclass(frozen=True)
class GridSpec:
    """grid.hpp:25-43."""
    kind: int
    nlat: int
    nlon: int
    colatitudes: np.ndarray = dc_field(repr=False, compare=False)
    longitudes: np.ndarray = dc_field(repr=False, compare=False)
    quad_weights: np.ndarray = dc_field(repr=False, compare=False)

    def same_sampling(self, o: "GridSpec") -> bool:
        return self.kind == o.kind and self.nlat == o.nlat and self.nlon == o.nlon

    def total_weight(self) -> float:
        return float(self.quad_weights.sum() * self.nlon)


def _grid(kind: int, nlat: int, nlon: int) -> GridSpec:
    c = np.zeros(max(nlat, 1))
    w = np.zeros(max(nlat, 1))
    check(L.lib.sph_grid(kind, nlat, nlon, c.ctypes.data_as(C.POINTER(C.c_double)),
                         w.ctypes.data_as(C.POINTER(C.c_double))))
    lon = 2.0 * PI * np.arange(nlon, dtype=np.float64) / nlon
    return GridSpec(kind, nlat, nlon, c[:nlat], lon, w[:nlat])


def build_equiangular(nlat: int, nlon: int) -> GridSpec:
    """grid.hpp:69-87: theta_i = pi i / nlat (north-pole row included)."""
    return _grid(EQUIANGULAR, nlat, nlon)


def build_gaussian(nlat: int, nlon: int) -> GridSpec:
    """grid.hpp:91-128: Gauss-Legendre nodes in cos(theta)."""
    return _grid(GAUSSIAN, nlat, nlon)


def default_mmax(lmax: int, nlon: int) -> int:
    """harmonics.hpp:120-122."""
    return min(lmax, nlon // 2 + 1)


# ------------------------------------------------------------------ fields
@dataclass
class SphericalField:
    """field.hpp:15-35; data [..., channels, nlat, nlon] fp32 on a CUDA device."""
    grid: GridSpec
    data: torch.Tensor

    @property
    def channels(self) -> int:
        return int(self.data.shape[-3])

    def npoints(self) -> int:
        return self.grid.nlat * self.grid.nlon


@dataclass
class SpectralCoeffs:
    """harmonics.hpp:24-42; coeffs [..., channels, lmax, mmax] complex64."""
    lmax: int
    mmax: int
    coeffs: torch.Tensor

    @property
    def channels(self) -> int:
        return int(self.coeffs.shape[-3])


def require_same_sampling(f: SphericalField, g: GridSpec, where: str) -> None:
    """field.hpp:37-43."""
    if not f.grid.same_sampling(g):
        raise L.SphInvalidArgument(1, f"{where}: grid/field shape mismatch")
    if tuple(f.data.shape[-2:]) != (g.nlat, g.nlon):
        raise L.SphInvalidArgument(1, f"{where}: field storage inconsistent")


def _stream(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _dev_f32(t: torch.Tensor, what: str) -> torch.Tensor:
    if not t.is_cuda:
        raise L.SphInvalidArgument(1, f"{what}: tensor must live on a CUDA device")
    return t.to(torch.float32).contiguous()


# -------------------------------------------------------------------- plans
_plan_lock = threading.Lock()
_sht_plans: dict = {}
_disco_plans: dict = {}


class ShtPlan:
    """One-time host precompute + device tables for (grid, lmax, mmax): replaces the
    per-call table builds of harmonics.hpp:159-162 / :202-205."""

    def __init__(self, grid: GridSpec, lmax: int, mmax: int, precision: str = "3xtf32",
                 allow_equiangular_forward: bool = False, device=None, adjoint: bool = False):
        self.grid, self.lmax, self.mmax = grid, int(lmax), int(mmax)
        self.device = torch.device("cuda", _dev_index(device))
        flags = PRECISIONS[precision] | (L.SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD
                                         if allow_equiangular_forward else 0)
        if adjoint:  # forward / inverse compute the adjoints of inverse / forward
            flags |= L.SPH_FLAG_ADJOINT
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(L.lib.sph_sht_plan_create(grid.kind, grid.nlat, grid.nlon, self.lmax,
                                            self.mmax, flags, C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and L is not None and L.lib is not None:
            L.lib.sph_sht_plan_destroy(h)
            self.h = None

    # sizes
    def coeffs_elems(self, F: int, layout: int) -> int:
        return int(L.lib.sph_sht_coeffs_elems(self.h, F, layout))

    def workspace(self, F: int) -> torch.Tensor:
        n = int(L.lib.sph_sht_workspace_bytes(self.h, F))
        return torch.empty(n, dtype=torch.uint8, device=self.device)

    # raw tensor entry points: x [F, nlat, nlon] -> coeffs
    def forward(self, x: torch.Tensor, layout: int = L.SPH_LAYOUT_DENSE_LM, out=None, ws=None):
        g = self.grid
        x = _dev_f32(x, "sht_forward")
        F = x.numel() // (g.nlat * g.nlon)
        if out is None:
            if layout == L.SPH_LAYOUT_DENSE_LM:
                out = torch.empty((F, self.lmax, self.mmax, 2), dtype=torch.float32, device=x.device)
            else:  # padding beyond each (m, parity) block stays zero
                out = torch.zeros(self.coeffs_elems(F, layout), dtype=torch.float32, device=x.device)
        ws = self.workspace(F) if ws is None else ws
        check(L.lib.sph_sht_forward(self.h, _ptr(x), F, _ptr(out), layout, _ptr(ws),
                                    _stream(x.device)))
        return out

    def inverse(self, coeffs: torch.Tensor, F: int, layout: int = L.SPH_LAYOUT_DENSE_LM,
                out=None, ws=None):
        g = self.grid
        if coeffs.dtype == torch.complex64:
            coeffs = torch.view_as_real(coeffs.contiguous())
        coeffs = _dev_f32(coeffs, "sht_inverse")
        if out is None:
            out = torch.empty((F, g.nlat, g.nlon), dtype=torch.float32, device=coeffs.device)
        ws = self.workspace(F) if ws is None else ws
        check(L.lib.sph_sht_inverse(self.h, _ptr(coeffs), F, layout, _ptr(out), _ptr(ws),
                                    _stream(coeffs.device)))
        return out

    def roundtrip_host(self, x_host: torch.Tensor, y_host: torch.Tensor, chunk: int = 32):
        """sht_inverse(sht_forward(x)) for host buffers, H2D/compute/D2H pipelined."""
        F = x_host.numel() // (self.grid.nlat * self.grid.nlon)
        with torch.cuda.device(self.device):
            check(L.lib.sph_sht_roundtrip_host(self.h, _ptr(x_host), F, _ptr(y_host), chunk))

    # distributed stages (distsim.hpp:413-430, :437-459)
    def fft_stage(self, rings: torch.Tensor, F: int, h_count: int, out=None):
        if out is None:
            out = torch.empty((F, h_count, self.mmax, 2), dtype=torch.float32, device=rings.device)
        check(L.lib.sph_sht_fft_stage(self.h, _ptr(rings), F, h_count, _ptr(out),
                                      _stream(rings.device)))
        return out

    def legendre_stage(self, bins: torch.Tensor, F: int, m0: int, m_count: int, out=None):
        if out is None:
            out = torch.empty((F, self.lmax, m_count, 2), dtype=torch.float32, device=bins.device)
        n = int(L.lib.sph_sht_stage_workspace_bytes(self.h, F, m_count))
        ws = torch.empty(n, dtype=torch.uint8, device=bins.device)
        check(L.lib.sph_sht_legendre_stage(self.h, _ptr(bins), F, m0, m_count, _ptr(out),
                                           _ptr(ws), _stream(bins.device)))
        return out


def _dev_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    return torch.cuda.current_device() if d.index is None else d.index


def get_sht_plan(grid: GridSpec, lmax: int, mmax: int, precision: str = "3xtf32",
                 allow_equiangular_forward: bool = False, adjoint: bool = False, device=None) -> ShtPlan:
    """Plan cache keyed by the device of the data (``device``, default the current one):
    a tensor on cuda:1 gets a cuda:1 plan whatever device is current."""
    dev = _dev_index(device)
    key = (grid.kind, grid.nlat, grid.nlon, lmax, mmax, precision, allow_equiangular_forward, dev, adjoint)
    with _plan_lock:
        p = _sht_plans.get(key)
        if p is None:
            p = ShtPlan(grid, lmax, mmax, precision, allow_equiangular_forward, device=dev, adjoint=adjoint)
            _sht_plans[key] = p
        return p


# --------------------------------------------------------------------- SHT
def sht_forward(field: SphericalField, lmax: Optional[int] = None, mmax: Optional[int] = None,
                precision: str = "3xtf32") -> SpectralCoeffs:
    """harmonics.hpp:126-169.  Gaussian grids only: the reference throws
    std::invalid_argument on equiangular grids (harmonics.hpp:129-130); its equiangular
    forward path is dist_sht_forward (see paper_2507_12144_b200.dist)."""
    g = field.grid
    if lmax is None:  # harmonics.hpp:164-169
        lmax = g.nlat
        mmax = max(min(default_mmax(lmax, g.nlon), g.nlon // 2), 1)
    elif mmax is None:
        raise L.SphInvalidArgument(1, "sht_forward: give both lmax and mmax")
    if g.kind != GAUSSIAN:
        raise L.SphInvalidArgument(1, "sht_forward: requires a gaussian grid")
    if g.nlat < lmax or g.nlon < 2 * mmax:
        raise L.SphInvalidArgument(1, "sht_forward: resolution insufficient for lmax/mmax")
    if mmax > lmax:
        raise L.SphInvalidArgument(1, "SpectralCoeffs: mmax must be <= lmax")
    return _forward(field, lmax, mmax, precision, allow_eq=False)


def _forward(field: SphericalField, lmax: int, mmax: int, precision: str,
             allow_eq: bool) -> SpectralCoeffs:
    g = field.grid
    lead = tuple(field.data.shape[:-2])
    plan = get_sht_plan(g, lmax, mmax, precision, allow_eq, device=field.data.device)
    with torch.cuda.device(field.data.device):
        out = plan.forward(field.data)
    return SpectralCoeffs(lmax, mmax, torch.view_as_complex(out).reshape(*lead, lmax, mmax))


def sht_inverse(coeffs: SpectralCoeffs, grid: GridSpec,
                precision: str = "3xtf32") -> SphericalField:
    """harmonics.hpp:173-205 (any grid kind)."""
    if coeffs.mmax > coeffs.lmax:
        raise L.SphInvalidArgument(1, "SpectralCoeffs: mmax must be <= lmax")
    c = coeffs.coeffs
    lead = tuple(c.shape[:-2])
    F = int(np.prod(lead)) if lead else 1
    plan = get_sht_plan(grid, coeffs.lmax, coeffs.mmax, precision, device=c.device)
    with torch.cuda.device(c.device):
        y = plan.inverse(c.to(torch.complex64), F)
    return SphericalField(grid, y.reshape(*lead, grid.nlat, grid.nlon))


# ----------------------------------------------------------- SHT adjoints
# The SHT's backward pass ("SHT adjoints come next"; the reference has no
# counterpart).  Inner products: sum Re(conj(c) d) over the stored m >= 0 coefficients and
# the plain sum over grid samples; pinned by the adjoint identities (tests/test_sht_gpu.py)
# and by the fp64 oracle restatement of the same formulas (tests/test_oracle.py).
def sht_forward_adjoint(coeffs: SpectralCoeffs, grid: GridSpec, precision: str = "3xtf32") -> SphericalField:
    """Adjoint of sht_forward on ``grid`` (Gaussian): coefficients [..., lmax, mmax] ->
    field, y_ij = w_i * sum_lm P_lm(theta_i) Re(d_lm e^{i m phi_j})."""
    if grid.kind != GAUSSIAN:
        raise L.SphInvalidArgument(1, "sht_forward: requires a gaussian grid")
    c = coeffs.coeffs
    lead = tuple(c.shape[:-2])
    F = int(np.prod(lead)) if lead else 1
    plan = get_sht_plan(grid, coeffs.lmax, coeffs.mmax, precision, adjoint=True, device=c.device)
    with torch.cuda.device(c.device):
        y = plan.inverse(c.to(torch.complex64), F)
    return SphericalField(grid, y.reshape(*lead, grid.nlat, grid.nlon))


def sht_inverse_adjoint(field: SphericalField, lmax: int, mmax: int, precision: str = "3xtf32") -> SpectralCoeffs:
    """Adjoint of sht_inverse(., field.grid) for (lmax, mmax) coefficients: field ->
    coefficients c_lm = (m ? 2 : 1) sum_ij P_lm(theta_i) z_ij e^{-i m phi_j} (any grid kind)."""
    g = field.grid
    if g.nlat < lmax or g.nlon < 2 * mmax:
        raise L.SphInvalidArgument(1, "sht_forward: resolution insufficient for lmax/mmax")
    if mmax > lmax:
        raise L.SphInvalidArgument(1, "SpectralCoeffs: mmax must be <= lmax")
    lead = tuple(field.data.shape[:-2])
    plan = get_sht_plan(g, lmax, mmax, precision, adjoint=True, device=field.data.device)
    with torch.cuda.device(field.data.device):
        out = plan.forward(field.data)
    return SpectralCoeffs(lmax, mmax, torch.view_as_complex(out).reshape(*lead, lmax, mmax))


# ------------------------------------------------------------------- DISCO
@dataclass(frozen=True)
class FilterBasis:
    """convolution.hpp:30-69."""
    theta_cutoff: float
    indices: tuple
    kind: int

    def n_pairs(self) -> int:
        return len(self.indices)

    def n_real(self) -> int:
        return sum(1 if p == (0, 0) else 2 for p in self.indices)


def morlet_basis(theta_cutoff: float) -> FilterBasis:
    """convolution.hpp:73-76 (K = 9)."""
    if theta_cutoff <= 0.0:
        raise L.SphInvalidArgument(1, "morlet_basis: cutoff must be > 0")
    return FilterBasis(float(theta_cutoff), ((0, 0), (0, 1), (0, 2), (2, 1), (2, 2)),
                       L.SPH_BASIS_MORLET)


def isotropic_basis(theta_cutoff: float) -> FilterBasis:
    """convolution.hpp:78-81 (K = 1)."""
    if theta_cutoff <= 0.0:
        raise L.SphInvalidArgument(1, "isotropic_basis: cutoff must be > 0")
    return FilterBasis(float(theta_cutoff), ((0, 0),), L.SPH_BASIS_ISOTROPIC)


class DiscoOperator:
    """convolution.hpp:105-123: the assembled operator lives on the device."""

    def __init__(self, in_grid: GridSpec, out_grid: GridSpec, basis: FilterBasis,
                 precision: str = "3xtf32", device=None):
        self.in_grid, self.out_grid, self.basis = in_grid, out_grid, basis
        self.device = torch.device("cuda", _dev_index(device))
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(L.lib.sph_disco_plan_create(in_grid.kind, in_grid.nlat, in_grid.nlon,
                                              out_grid.kind, out_grid.nlat, out_grid.nlon,
                                              basis.kind, basis.theta_cutoff, PRECISIONS[precision],
                                              C.byref(h)))
        self.h = h
        k, s, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        check(L.lib.sph_disco_plan_info(h, C.byref(k), C.byref(s), C.byref(nnz)))
        self.n_basis, self.stride, self.nnz_per_basis = k.value, s.value, nnz.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and L is not None and L.lib is not None:
            L.lib.sph_disco_plan_destroy(h)
            self.h = None

    def workspace(self, B: int, cin: int, cout: int) -> torch.Tensor:
        n = int(L.lib.sph_disco_workspace_bytes(self.h, B, cin, cout))
        return torch.empty(n, dtype=torch.uint8, device=self.device)

    def apply(self, x: torch.Tensor, mix: torch.Tensor, out=None, ws=None) -> torch.Tensor:
        """x [B, cin, hin, win] -> y [B, cout, hout, wout]."""
        mix = _dev_f32(mix, "disco_apply")
        x = _dev_f32(x, "disco_apply")
        cout, cin, K = mix.shape
        if K != self.n_basis or x.shape[-3] != cin:
            raise L.SphInvalidArgument(1, "disco_apply: mix tensor shape mismatch")
        B = x.numel() // (cin * self.in_grid.nlat * self.in_grid.nlon)
        if out is None:
            out = torch.empty((B, cout, self.out_grid.nlat, self.out_grid.nlon),
                              dtype=torch.float32, device=x.device)
        ws = self.workspace(B, cin, cout) if ws is None else ws
        check(L.lib.sph_disco_apply(self.h, _ptr(x), _ptr(mix), B, cin, cout, _ptr(out),
                                    _ptr(ws), _stream(x.device)))
        return out


    def transpose_apply(self, v: torch.Tensor, mix: torch.Tensor, out=None, ws=None) -> torch.Tensor:
        """disco_transpose_apply (convolution.hpp:226-266): v [B, cout, hout, wout] on the
        output grid -> [B, cin, hin, win] on the input grid; ``mix`` is the forward's
        [cout, cin, K] tensor."""
        mix = _dev_f32(mix, "disco_transpose_apply")
        v = _dev_f32(v, "disco_transpose_apply")
        cout, cin, K = mix.shape
        if K != self.n_basis or v.shape[-3] != cout:
            raise L.SphInvalidArgument(1, "disco_transpose_apply: mix tensor shape mismatch")
        if v.shape[-2:] != (self.out_grid.nlat, self.out_grid.nlon):
            raise L.SphInvalidArgument(1, "disco_transpose_apply: field sampling mismatch")
        B = v.numel() // (cout * self.out_grid.nlat * self.out_grid.nlon)
        if out is None:
            out = torch.empty((B, cin, self.in_grid.nlat, self.in_grid.nlon),
                              dtype=torch.float32, device=v.device)
        if ws is None:
            n = L.lib.sph_disco_transpose_workspace_bytes(self.h, B, cin, cout)
            ws = torch.empty(max(n, 1), dtype=torch.uint8, device=v.device)
        check(L.lib.sph_disco_transpose_apply(self.h, _ptr(v), _ptr(mix), B, cin, cout, _ptr(out),
                                              _ptr(ws), _stream(v.device)))
        return out

    def input_rows(self, ho0: int, nout: int):
        """Input latitude rows (h_in0, n_in) covering the filter support of output rows
        [ho0, ho0 + nout) -- the halo a latitude shard needs."""
        lo, n = C.c_int64(), C.c_int64()
        check(L.lib.sph_disco_input_rows(self.h, ho0, nout, C.byref(lo), C.byref(n)))
        return lo.value, n.value

    def apply_rows(self, x: torch.Tensor, h_in0: int, ho0: int, nout: int, mix: torch.Tensor,
                   out=None) -> torch.Tensor:
        """Latitude-shard apply: x [B, cin, nin, win] holds input rows [h_in0, h_in0+nin);
        returns output rows [ho0, ho0+nout) as [B, cout, nout, wout]."""
        mix = _dev_f32(mix, "disco_apply")
        x = _dev_f32(x, "disco_apply")
        cout, cin, K = mix.shape
        if K != self.n_basis or x.shape[-3] != cin:
            raise L.SphInvalidArgument(1, "disco_apply: mix tensor shape mismatch")
        B, nin = x.shape[0], x.shape[-2]
        if out is None:
            out = torch.empty((B, cout, nout, self.out_grid.nlon), dtype=torch.float32, device=x.device)
        n = int(L.lib.sph_disco_rows_workspace_bytes(self.h, B, cin, cout, nin, nout))
        ws = torch.empty(n, dtype=torch.uint8, device=x.device)
        check(L.lib.sph_disco_apply_rows(self.h, _ptr(x), h_in0, nin, ho0, nout, _ptr(mix), B, cin,
                                         cout, _ptr(out), _ptr(ws), _stream(x.device)))
        return out


def assemble_disco(in_grid: GridSpec, out_grid: GridSpec, basis: FilterBasis,
                   precision: str = "3xtf32", device=None) -> DiscoOperator:
    """convolution.hpp:141-177 (the operator lives on ``device``, default the current one)."""
    dev = _dev_index(device)
    key = (in_grid.kind, in_grid.nlat, in_grid.nlon, out_grid.kind, out_grid.nlat,
           out_grid.nlon, basis, precision, dev)
    with _plan_lock:
        op = _disco_plans.get(key)
    if op is None:
        op = DiscoOperator(in_grid, out_grid, basis, precision, device=dev)
        with _plan_lock:
            _disco_plans[key] = op
    return op


def disco_apply(op: DiscoOperator, field: SphericalField, mix: torch.Tensor) -> SphericalField:
    """convolution.hpp:181-220: y[o] = sum_{c,k} mix[o,c,k] (psi_k * u_c)."""
    require_same_sampling(field, op.in_grid, "disco_apply")
    if mix.shape[1] != field.channels or mix.shape[2] != op.n_basis:
        raise L.SphInvalidArgument(1, "disco_apply: mix tensor shape mismatch")
    lead = tuple(field.data.shape[:-3])
    with torch.cuda.device(field.data.device):
        y = op.apply(field.data, mix)
    return SphericalField(op.out_grid, y.reshape(*lead, mix.shape[0], op.out_grid.nlat,
                                                  op.out_grid.nlon))


def disco_transpose_apply(op: DiscoOperator, field: SphericalField, mix: torch.Tensor) -> SphericalField:
    """convolution.hpp:226-266: the adjoint of disco_apply under the quadrature inner
    products; ``field`` lives on the output grid, the result on the input grid."""
    require_same_sampling(field, op.out_grid, "disco_transpose_apply")
    if mix.shape[0] != field.channels or mix.shape[2] != op.n_basis or mix.shape[1] == 0:
        raise L.SphInvalidArgument(1, "disco_transpose_apply: mix tensor shape mismatch")
    lead = tuple(field.data.shape[:-3])
    with torch.cuda.device(field.data.device):
        y = op.transpose_apply(field.data, mix)
    return SphericalField(op.in_grid, y.reshape(*lead, mix.shape[1], op.in_grid.nlat,
                                                 op.in_grid.nlon))


# ------------------------------------------------------------------ resample
_RESAMPLE_PLANS: Dict[tuple, "ResamplePlan"] = {}


class ResamplePlan:
    """bilinear_resample tables (resample.hpp:66-114) for one (input grid, output grid)
    pair: fp64 brackets / weights built once on the host, device gather per call."""

    def __init__(self, in_grid: GridSpec, out_grid: GridSpec):
        self.in_grid, self.out_grid = in_grid, out_grid
        ci = np.ascontiguousarray(in_grid.colatitudes, dtype=np.float64)
        co = np.ascontiguousarray(out_grid.colatitudes, dtype=np.float64)
        h = C.c_void_p()
        check(L.lib.sph_resample_plan_create(ci.ctypes.data, in_grid.nlat, in_grid.nlon, co.ctypes.data,
                                             out_grid.nlat, out_grid.nlon, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and L.lib is not None:
            L.lib.sph_resample_plan_destroy(self.h)

    def apply(self, x: torch.Tensor, out=None) -> torch.Tensor:
        x = _dev_f32(x, "bilinear_resample")
        gi, go = self.in_grid, self.out_grid
        if tuple(x.shape[-2:]) != (gi.nlat, gi.nlon):
            raise L.SphInvalidArgument(1, "bilinear_resample: field sampling mismatch")
        Cn = x.numel() // (gi.nlat * gi.nlon)
        if out is None:
            out = torch.empty(tuple(x.shape[:-2]) + (go.nlat, go.nlon), dtype=torch.float32, device=x.device)
        ws = torch.empty(max(1, int(L.lib.sph_resample_workspace_bytes(self.h, Cn))), dtype=torch.uint8,
                         device=x.device)
        with torch.cuda.device(x.device):
            check(L.lib.sph_bilinear_resample(self.h, _ptr(x), Cn, _ptr(out), _ptr(ws), _stream(x.device)))
        return out


def bilinear_resample(field: SphericalField, out_grid: GridSpec) -> SphericalField:
    """resample.hpp:66-114: four-weight bilinear interpolation with pole extension."""
    key = (field.grid.kind, field.grid.nlat, field.grid.nlon, tuple(np.asarray(field.grid.colatitudes)[[0, -1]]),
           out_grid.kind, out_grid.nlat, out_grid.nlon)
    plan = _RESAMPLE_PLANS.get(key)
    if plan is None:
        plan = _RESAMPLE_PLANS[key] = ResamplePlan(field.grid, out_grid)
    return SphericalField(out_grid, plan.apply(field.data))


def spectral_resample(field: SphericalField, out_grid: GridSpec, precision: str = "3xtf32") -> SphericalField:
    """resample.hpp:120-132: alias-free resampling, forward SHT truncated to the smaller
    grid's capacity then synthesis on ``out_grid``; non-Gaussian inputs are first moved
    to the Gaussian grid of the same size by bilinear interpolation."""
    src = field
    if field.grid.kind != GAUSSIAN:
        src = bilinear_resample(field, build_gaussian(field.grid.nlat, field.grid.nlon))
    lmax = min(src.grid.nlat, out_grid.nlat)
    mmax = min(lmax, src.grid.nlon // 2, (out_grid.nlon - 1) // 2 + 1)
    return sht_inverse(sht_forward(src, lmax, mmax, precision), out_grid, precision)


# ------------------------------------------------------------------ decoder
class DecoderPlan:
    """decode_preclamp's per-group body (model.hpp:372-394): disco_apply(op,
    bilinear_resample(latent, op.in_grid), mix) with the upsampling applied to the latent's
    ring spectra inside the convolution when op.in_grid.nlon is a multiple of the latent's."""

    def __init__(self, op: DiscoOperator, latent_grid: GridSpec):
        if (op.in_grid.kind, op.in_grid.nlat, op.in_grid.nlon) != (op.out_grid.kind, op.out_grid.nlat,
                                                                    op.out_grid.nlon):
            raise L.SphInvalidArgument(1, "decode: the decoder convolution maps the output grid onto itself")
        self.op, self.latent_grid = op, latent_grid
        ci = np.ascontiguousarray(latent_grid.colatitudes, dtype=np.float64)
        h = C.c_void_p()
        check(L.lib.sph_decoder_plan_create(op.h, ci.ctypes.data, latent_grid.nlat, latent_grid.nlon, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and L.lib is not None:
            L.lib.sph_decoder_plan_destroy(self.h)
            self.h = None

    def apply(self, latent: torch.Tensor, mix: torch.Tensor, out=None, ws=None) -> torch.Tensor:
        """latent [B, cin, latent_nlat, latent_nlon] -> y [B, cout, out_nlat, out_nlon]."""
        mix = _dev_f32(mix, "decode")
        latent = _dev_f32(latent, "decode")
        cout, cin, K = mix.shape
        gl, go = self.latent_grid, self.op.out_grid
        if K != self.op.n_basis or latent.shape[-3] != cin:
            raise L.SphInvalidArgument(1, "decode: mix tensor shape mismatch")
        if tuple(latent.shape[-2:]) != (gl.nlat, gl.nlon):
            raise L.SphInvalidArgument(1, "decode: latent sampling mismatch")
        B = latent.numel() // (cin * gl.nlat * gl.nlon)
        if out is None:
            out = torch.empty((B, cout, go.nlat, go.nlon), dtype=torch.float32, device=latent.device)
        if ws is None:
            ws = torch.empty(int(L.lib.sph_decoder_workspace_bytes(self.h, B, cin, cout)), dtype=torch.uint8,
                             device=latent.device)
        with torch.cuda.device(latent.device):
            check(L.lib.sph_decoder_apply(self.h, _ptr(latent), _ptr(mix), B, cin, cout, _ptr(out), _ptr(ws),
                                          _stream(latent.device)))
        return out


_DECODER_PLANS: Dict[tuple, DecoderPlan] = {}


def decode_preclamp(op: DiscoOperator, latent: SphericalField, mixes) -> SphericalField:
    """model.hpp:372-394: the latent channels split into consecutive groups, group g of
    mixes[g].shape[1] channels decoded by disco_apply(op, upsampled group, mixes[g]); the
    outputs are concatenated along channels.  Upsampling and convolution run fused."""
    if isinstance(mixes, torch.Tensor) and mixes.dim() == 3:
        mixes = [mixes]
    key = (id(op), latent.grid.kind, latent.grid.nlat, latent.grid.nlon,
           tuple(np.asarray(latent.grid.colatitudes)[[0, -1]]))
    plan = _DECODER_PLANS.get(key)
    if plan is None or plan.op is not op:
        plan = _DECODER_PLANS[key] = DecoderPlan(op, latent.grid)
    x = latent.data
    if sum(int(m.shape[1]) for m in mixes) != x.shape[-3]:
        raise L.SphInvalidArgument(1, "decode: channel groups do not cover the latent channels")
    lead = tuple(x.shape[:-3])
    x = x.reshape(-1, *x.shape[-3:])
    outs, c0 = [], 0
    for m in mixes:
        cin = int(m.shape[1])
        outs.append(plan.apply(x[:, c0:c0 + cin].contiguous(), m))
        c0 += cin
    y = torch.cat(outs, dim=1)
    return SphericalField(op.out_grid, y.reshape(*lead, y.shape[1], op.out_grid.nlat, op.out_grid.nlon))


# ------------------------------------------------------------ SHT consumers
CRPS_VARIANTS = {"cdf": 0, "spread_skill": 1, "fair": 2}


def angular_psd(field: SphericalField, precision: str = "3xtf32") -> torch.Tensor:
    """metrics.hpp:300-314: PSD(l) = sum_{|m|<=l} |uhat_l^m|^2 per channel, lmax = nlat
    (Gaussian grids only, through sht_forward like the reference).  Returns [..., C, nlat]."""
    g = field.grid
    if g.kind != GAUSSIAN:
        raise L.SphInvalidArgument(1, "sht_forward: requires a gaussian grid")
    lmax = g.nlat
    mmax = max(min(default_mmax(lmax, g.nlon), g.nlon // 2), 1)
    x = _dev_f32(field.data, "angular_psd")
    plan = get_sht_plan(g, lmax, mmax, precision, device=x.device)
    F = x.numel() // (g.nlat * g.nlon)
    with torch.cuda.device(x.device):
        c = plan.forward(x, L.SPH_LAYOUT_DENSE_LM)
        psd = torch.empty((F, lmax), dtype=torch.float32, device=x.device)
        check(L.lib.sph_psd_from_coeffs(_ptr(c), F, lmax, mmax, _ptr(psd), _stream(x.device)))
    return psd.reshape(tuple(x.shape[:-2]) + (lmax,))


def spectral_crps_loss(ens: torch.Tensor, obs: SphericalField, lmax_sum: int = 0,
                       variant: str = "spread_skill", precision: str = "3xtf32") -> torch.Tensor:
    """loss.hpp:37-81: ens [E][C][H][W] members on obs.grid (Gaussian), obs [C][H][W];
    sum over 1 <= l <= lmax_sum and stored orders of the CRPS of Re and Im, per channel
    (fp64 [C])."""
    g = obs.grid
    if g.kind != GAUSSIAN:
        raise L.SphInvalidArgument(1, "spectral_crps_loss: requires a gaussian grid")
    E, Cc = ens.shape[0], ens.shape[1]
    if tuple(ens.shape[2:]) != (g.nlat, g.nlon) or obs.channels != Cc:
        raise L.SphInvalidArgument(1, "spectral_crps_loss: shape mismatch")
    if lmax_sum == 0:
        lmax_sum = g.nlat // 2
    if lmax_sum + 1 > g.nlat:
        raise L.SphInvalidArgument(1, "spectral_crps_loss: lmax_sum exceeds grid capacity")
    lmax = lmax_sum + 1
    mmax = min(lmax, g.nlon // 2)
    ens = _dev_f32(ens, "spectral_crps_loss")
    plan = get_sht_plan(g, lmax, mmax, precision, device=ens.device)
    o = _dev_f32(obs.data, "spectral_crps_loss")
    with torch.cuda.device(ens.device):
        ce = plan.forward(ens.reshape(E * Cc, g.nlat, g.nlon), L.SPH_LAYOUT_DENSE_LM)
        co = plan.forward(o.reshape(Cc, g.nlat, g.nlon), L.SPH_LAYOUT_DENSE_LM)
        out = torch.empty(Cc, dtype=torch.float64, device=ens.device)
        check(L.lib.sph_spectral_crps_from_coeffs(_ptr(ce), _ptr(co), E, Cc, lmax, mmax, lmax_sum,
                                                  CRPS_VARIANTS[variant], _ptr(out), _stream(ens.device)))
    return out


# ----------------------------------------------------------- spectral conv
def spectral_conv(field: SphericalField, kernel: torch.Tensor,
                  precision: str = "3xtf32") -> SphericalField:
    """convolution.hpp:286-304; kernel [c_out][c_in][klmax]."""
    g = field.grid
    if g.kind != GAUSSIAN:
        raise L.SphInvalidArgument(1, "spectral_conv: requires a gaussian grid")
    cout, cin, klmax = kernel.shape
    if cin != field.channels:
        raise L.SphInvalidArgument(1, "spectral_conv: kernel channel mismatch")
    lmax = min(klmax, g.nlat)
    mmax = min(lmax, g.nlon // 2)
    x = _dev_f32(field.data, "spectral_conv")
    plan = get_sht_plan(g, lmax, mmax, precision, device=x.device)
    lead = tuple(x.shape[:-3])
    B = x.numel() // (cin * g.nlat * g.nlon)
    kernel = _dev_f32(kernel, "spectral_conv")
    y = torch.empty((B, cout, g.nlat, g.nlon), dtype=torch.float32, device=x.device)
    n = int(L.lib.sph_spectral_conv_workspace_bytes(plan.h, B, cin, cout))
    ws = torch.empty(n, dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        check(L.lib.sph_spectral_conv(plan.h, _ptr(x), _ptr(kernel), B, cin, cout, klmax,
                                      _ptr(y), _ptr(ws), _stream(x.device)))
    return SphericalField(g, y.reshape(*lead, cout, g.nlat, g.nlon))


def spectral_mix(coeffs: SpectralCoeffs, kernel: torch.Tensor, precision: str = "3xtf32",
                 grid: Optional[GridSpec] = None) -> SpectralCoeffs:
    """The channel mix of spectral_conv alone (convolution.hpp:295-302):
    out(.., o, l, m) = sum_i coeffs(.., i, l, m) kernel(o, i, l); coeffs [B][c_in][lmax][mmax]
    complex, kernel [c_out][c_in][klmax] with klmax >= lmax.  ``grid`` only selects the
    plan the mix runs on (any grid with nlat >= lmax, nlon >= 2 mmax)."""
    c = coeffs.coeffs
    if c.dtype != torch.complex64:
        c = c.to(torch.complex64)
    cout, cin, klmax = kernel.shape
    if c.shape[-3] != cin:
        raise L.SphInvalidArgument(1, "spectral_mix: kernel channel mismatch")
    lead = tuple(c.shape[:-3])
    B = int(np.prod(lead)) if lead else 1
    g = grid or build_gaussian(coeffs.lmax, max(2 * coeffs.mmax, 2))
    plan = get_sht_plan(g, coeffs.lmax, coeffs.mmax, precision, device=c.device)
    cr = torch.view_as_real(c.contiguous())
    k = _dev_f32(kernel, "spectral_mix")
    out = torch.empty((B, cout, coeffs.lmax, coeffs.mmax, 2), dtype=torch.float32, device=c.device)
    n = int(L.lib.sph_spectral_conv_workspace_bytes(plan.h, B, cin, cout))
    ws = torch.empty(n, dtype=torch.uint8, device=c.device)
    with torch.cuda.device(c.device):
        check(L.lib.sph_spectral_mix(plan.h, _ptr(cr), _ptr(k), B, cin, cout, klmax, _ptr(out), _ptr(ws),
                                     _stream(c.device)))
    return SpectralCoeffs(coeffs.lmax, coeffs.mmax,
                          torch.view_as_complex(out).reshape(*lead, cout, coeffs.lmax, coeffs.mmax))


# ------------------------------------------------------------------- block
@dataclass
class BlockWeights:
    """model.hpp:108-115 (one processor block)."""
    global_: bool
    conv: torch.Tensor        # mix [C][C+Cc][K] (local) or kernel [C][C+Cc][klmax] (global)
    w1: torch.Tensor          # [H][C]
    b1: torch.Tensor          # [H]
    w2: torch.Tensor          # [C][H]
    b2: torch.Tensor          # [C]
    scales: torch.Tensor      # [C]


def block_epilogue(conv: torch.Tensor, x: torch.Tensor, bw: BlockWeights) -> torch.Tensor:
    """model.hpp:355-368: y = x + scales * (W2 gelu(W1 gelu(conv) + b1) + b2)."""
    x = _dev_f32(x, "block_apply")
    conv = _dev_f32(conv, "block_apply")
    C_, H = bw.w2.shape
    P = x.shape[-1] * x.shape[-2]
    B = x.numel() // (C_ * P)
    y = torch.empty_like(x)
    w = [_dev_f32(t, "block_apply") for t in (bw.w1, bw.b1, bw.w2, bw.b2, bw.scales)]
    with torch.cuda.device(x.device):
        check(L.lib.sph_block_epilogue(_ptr(conv), _ptr(x), *[_ptr(t) for t in w], B, C_, H, P,
                                       _ptr(y), _stream(x.device)))
    return y


def block_apply(latent: SphericalField, conditioning: SphericalField, bw: BlockWeights,
                block_op: Optional[DiscoOperator] = None,
                precision: str = "3xtf32") -> SphericalField:
    """model.hpp:337-370: conv(concat(x, cond)) -> GeLU -> MLP -> layer-scaled residual.
    global blocks use spectral_conv, local blocks disco_apply with ``block_op``."""
    g = latent.grid
    require_same_sampling(latent, g, "block_apply")
    require_same_sampling(conditioning, g, "block_apply")
    cat = SphericalField(g, torch.cat([latent.data, conditioning.data], dim=-3))
    if bw.global_:
        conv = spectral_conv(cat, bw.conv, precision)
    else:
        if block_op is None:
            raise L.SphInvalidArgument(1, "block_apply: local block needs the block DISCO operator")
        conv = disco_apply(block_op, cat, bw.conv)
    return SphericalField(g, block_epilogue(conv.data, latent.data, bw).reshape(latent.data.shape))
