"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the spherical-operator hot path.

Two ctypes front ends over fp64 CPU code:

* ``orc``  -- the plain-C restatement in ``oracle/sphere_oracle.c`` (liboracle.so);
  every function there cites the reference file:line it restates.
* ``ref``  -- the UNMODIFIED reference headers (spheretk) compiled behind the C-ABI
  driver ``oracle/ref_driver.cpp`` into ``oracle/_ref/libsphref.so`` (only buildable
  where /root/reference exists; the built .so travels with the repo snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or the
reported CPU baseline.  The product (``paper_2507_12144_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libsphref.so")

EQUIANGULAR, GAUSSIAN = 0, 1
MORLET_PAIRS = [(0, 0), (0, 1), (0, 2), (2, 1), (2, 2)]  # convolution.hpp:73-76
ISOTROPIC_PAIRS = [(0, 0)]                                # convolution.hpp:78-81


def build() -> None:
    subprocess.run([os.path.join(HERE, "build.sh")], check=True)


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class OracleError(RuntimeError):
    pass


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------- restatement
class _Orc:
    def __init__(self):
        if not os.path.exists(_ORC_SO):
            build()
        L = C.CDLL(_ORC_SO)
        L.orc_grid.argtypes = [C.c_int, _sz, _sz, _dp, _dp]
        L.orc_legendre_table.argtypes = [_sz, _sz, _sz, _dp, _dp]
        L.orc_rfft_bins.argtypes = [_sz, _dp, _sz, _dp]
        L.orc_fft.argtypes = [_dp, _sz, C.c_int]
        L.orc_sht_forward.argtypes = [_sz, _sz, _dp, _dp, _sz, _sz, _sz, _dp, _dp]
        L.orc_sht_inverse.argtypes = [_sz, _sz, _dp, _sz, _sz, _sz, _dp, _dp]
        L.orc_disco_assemble.argtypes = [_sz, _sz, _dp, _dp, _sz, _sz, _dp,
                                         np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"),
                                         _sz, C.c_double, _i64p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        L.orc_disco_apply.argtypes = [_sz, _sz, _sz, _sz, _sz, _i64p, _i32p, _i32p, _dp,
                                      _sz, _sz, _dp, _dp, _dp]
        L.orc_disco_transpose_apply.argtypes = [_sz, _sz, _sz, _sz, _dp, _sz, _i64p, _i32p,
                                                _i32p, _dp, _sz, _sz, _dp, _dp, _dp]
        L.orc_spectral_conv.argtypes = [_sz, _sz, _dp, _dp, _sz, _sz, _sz, _dp, _dp, _dp]
        L.orc_random_uniform.argtypes = [C.c_uint64, _sz, _dp]
        L.orc_gelu.argtypes = [C.c_double]
        L.orc_gelu.restype = C.c_double
        L.orc_block_epilogue.argtypes = [_sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        self.L = L

    def random_uniform(self, shape, seed):
        """oracles.hpp:105-112 random_field stream (mt19937_64 + U(-1,1))."""
        out = np.zeros(int(np.prod(shape)))
        self.L.orc_random_uniform(seed, out.size, out)
        return out.reshape(shape)

    def grid(self, kind, nlat, nlon):
        colat = np.zeros(nlat)
        w = np.zeros(nlat)
        rc = self.L.orc_grid(kind, nlat, nlon, colat, w)
        if rc:
            raise OracleError(f"orc_grid rc={rc}")
        return colat, w

    def legendre_table(self, lmax, mmax, colat):
        colat = _c64(colat)
        out = np.zeros((len(colat), lmax, mmax))
        if self.L.orc_legendre_table(lmax, mmax, len(colat), colat, out):
            raise OracleError("legendre_table: mmax must be <= lmax")
        return out

    def rfft_bins(self, x, nbins):
        x = _c64(x)
        out = np.zeros(2 * nbins)
        self.L.orc_rfft_bins(len(x), x, nbins, out)
        return out[0::2] + 1j * out[1::2]

    def sht_forward(self, kind, nlat, nlon, lmax, mmax, x):
        """x [C][nlat][nlon] -> complex [C][lmax][mmax]; any grid kind."""
        x = _c64(x).reshape(-1, nlat, nlon)
        colat, w = self.grid(kind, nlat, nlon)
        out = np.zeros((x.shape[0], lmax, mmax, 2))
        if self.L.orc_sht_forward(nlat, nlon, colat, w, lmax, mmax, x.shape[0], x, out):
            raise OracleError("sht_forward: precondition")
        return out[..., 0] + 1j * out[..., 1]

    def sht_inverse(self, kind, nlat, nlon, coeffs):
        coeffs = np.asarray(coeffs)
        ch, lmax, mmax = coeffs.shape
        cf = np.ascontiguousarray(np.stack([coeffs.real, coeffs.imag], -1), dtype=np.float64)
        colat, _ = self.grid(kind, nlat, nlon)
        out = np.zeros((ch, nlat, nlon))
        if self.L.orc_sht_inverse(nlat, nlon, colat, lmax, mmax, ch, cf, out):
            raise OracleError("sht_inverse: precondition")
        return out

    def disco_assemble(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon,
                       cutoff, pairs=MORLET_PAIRS):
        ci, wi = self.grid(in_kind, in_nlat, in_nlon)
        co, _ = self.grid(out_kind, out_nlat, out_nlon)
        pr = np.ascontiguousarray(np.array(pairs, dtype=np.int32).reshape(-1))
        npairs = len(pairs)
        K = sum(1 if p == (0, 0) else 2 for p in pairs)  # convolution.hpp:59-63
        rp = np.zeros(out_nlat + 1, dtype=np.int64)
        rc = self.L.orc_disco_assemble(in_nlat, in_nlon, ci, wi, out_nlat, out_nlon, co, pr,
                                       npairs, cutoff, rp, None, None, None, None)
        if rc:
            raise OracleError(f"assemble_disco rc={rc}")
        n = int(rp[-1])
        h_in = np.zeros(n, dtype=np.int32)
        w_rel = np.zeros(n, dtype=np.int32)
        vals = np.zeros((n, K))
        base = np.zeros((n, K))
        rc = self.L.orc_disco_assemble(in_nlat, in_nlon, ci, wi, out_nlat, out_nlon, co, pr,
                                       npairs, cutoff, rp, h_in.ctypes.data, w_rel.ctypes.data,
                                       vals.ctypes.data, base.ctypes.data)
        assert rc == 0
        return dict(row_ptr=rp, h_in=h_in, w_rel=w_rel, vals=vals, base=base, K=K,
                    in_shape=(in_nlat, in_nlon), out_shape=(out_nlat, out_nlon),
                    out_weights=self.grid(out_kind, out_nlat, out_nlon)[1])

    def disco_apply(self, op, x, mix):
        (hi, wi), (ho, wo) = op["in_shape"], op["out_shape"]
        x = _c64(x).reshape(-1, hi, wi)
        mix = _c64(mix)
        cout, cin, K = mix.shape
        assert cin == x.shape[0] and K == op["K"]
        y = np.zeros((cout, ho, wo))
        self.L.orc_disco_apply(hi, wi, ho, wo, K, op["row_ptr"], op["h_in"], op["w_rel"],
                               _c64(op["vals"]), cin, cout, x, mix, y)
        return y

    def disco_transpose_apply(self, op, x, mix):
        (hi, wi), (ho, wo) = op["in_shape"], op["out_shape"]
        mix = _c64(mix)
        cout, cin, K = mix.shape
        x = _c64(x).reshape(cout, ho, wo)
        y = np.zeros((cin, hi, wi))
        self.L.orc_disco_transpose_apply(hi, wi, ho, wo, _c64(op["out_weights"]), K,
                                         op["row_ptr"], op["h_in"], op["w_rel"],
                                         _c64(op["base"]), cin, cout, x, mix, y)
        return y

    def spectral_conv(self, kind, nlat, nlon, kernel, x):
        kernel = _c64(kernel)
        cout, cin, klmax = kernel.shape
        x = _c64(x).reshape(cin, nlat, nlon)
        colat, w = self.grid(kind, nlat, nlon)
        y = np.zeros((cout, nlat, nlon))
        if self.L.orc_spectral_conv(nlat, nlon, colat, w, cin, cout, klmax, kernel, x, y):
            raise OracleError("spectral_conv")
        return y

    def block_epilogue(self, conv, x, w1, b1, w2, b2, scales):
        conv = _c64(conv)
        Cc = conv.shape[0]
        npts = conv[0].size
        H = len(b1)
        out = np.zeros(conv.shape)
        self.L.orc_block_epilogue(Cc, H, npts, conv, _c64(x), _c64(w1), _c64(b1), _c64(w2),
                                  _c64(b2), _c64(scales), out)
        return out

    def gelu(self, x):
        return self.L.orc_gelu(float(x))


# ----------------------------------------------------------------- reference
class _Ref:
    def __init__(self):
        if not os.path.exists(_REF_SO):
            build()
        if not os.path.exists(_REF_SO):
            raise OracleError("oracle/_ref/libsphref.so not built (needs /root/reference)")
        L = C.CDLL(_REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_uniform.argtypes = [C.c_ulonglong, _sz, _dp]
        L.ref_grid.argtypes = [C.c_int, _sz, _sz, _dp, _dp]
        L.ref_legendre_table.argtypes = [_sz, _sz, C.c_int, _sz, _sz, C.c_int, _dp]
        L.ref_rfft_bins.argtypes = [_sz, _dp, _sz, _dp]
        L.ref_sht_forward.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, _dp, _dp, C.c_int]
        L.ref_sht_inverse.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, _dp, _dp]
        L.ref_disco_rows.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int, C.c_double,
                                     np.ctypeslib.ndpointer(dtype=np.uint64), C.POINTER(_sz)]
        L.ref_disco_entries.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int,
                                        C.c_double, _i64p, _i64p, _dp, _dp]
        L.ref_disco_apply.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int, C.c_double,
                                      _sz, _sz, _dp, _dp, _dp]
        L.ref_disco_transpose_apply.argtypes = L.ref_disco_apply.argtypes
        L.ref_bilinear_resample.argtypes = [C.c_int, _sz, _sz, C.c_int, C.c_int, _sz, _sz, _sz, _dp, _dp]
        L.ref_spectral_resample.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, _sz, _dp, _dp]
        L.ref_angular_psd.argtypes = [C.c_int, _sz, _sz, _sz, _dp, _dp]
        L.ref_crps_field.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _dp, _dp, C.c_int, _dp]
        L.ref_write_sfd.argtypes = [C.c_char_p, C.c_int, _sz, _sz, _sz, _dp]
        L.ref_write_weights.argtypes = [C.c_char_p, _sz, _sz, _dp, _dp]
        L.ref_read_sfd.argtypes = [C.c_char_p, _dp, _sz, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz)]
        L.ref_noise_stream.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _dp, C.c_uint64, _sz, _dp, _dp]
        L.ref_spectral_crps_loss.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _dp, _dp, _sz, C.c_int, _dp]
        L.ref_spectral_conv.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, _dp, _dp, _dp]
        L.ref_block_apply.argtypes = [_sz, _sz, _sz, _sz, _sz, C.c_int, C.c_double, _sz, _dp,
                                      _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_block_channels.restype = _sz
        L.ref_block_channels.argtypes = [_sz, _sz]
        L.ref_dist_sht_forward.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _dp, _dp,
                                           C.c_char_p, _sz]
        L.ref_dist_disco_apply.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int,
                                           C.c_double, _sz, _sz, _sz, _sz, _dp, _dp, _dp,
                                           C.c_char_p, _sz]
        L.ref_bench_sht_roundtrip.argtypes = [C.c_int, _sz, _sz, _sz, _sz, _sz, _sz, _dp,
                                              C.c_void_p, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double)]
        L.ref_bench_disco.argtypes = [C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int, C.c_double,
                                      _sz, _sz, _sz, _dp, _dp, C.c_void_p,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self.L = L

    def _check(self, rc):
        if rc:
            msg = self.L.ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)       # std::invalid_argument
            raise RuntimeError(msg)         # std::runtime_error

    def random_uniform(self, shape, seed):
        out = np.zeros(int(np.prod(shape)))
        self.L.ref_random_uniform(seed, out.size, out)
        return out.reshape(shape)

    def grid(self, kind, nlat, nlon):
        colat = np.zeros(nlat)
        w = np.zeros(nlat)
        self._check(self.L.ref_grid(kind, nlat, nlon, colat, w))
        return colat, w

    def legendre_table(self, lmax, mmax, kind, nlat, nlon, weighted=False):
        out = np.zeros((nlat, lmax, mmax))
        self._check(self.L.ref_legendre_table(lmax, mmax, kind, nlat, nlon, int(weighted), out))
        return out

    def rfft_bins(self, x, nbins):
        x = _c64(x)
        out = np.zeros(2 * nbins)
        self._check(self.L.ref_rfft_bins(len(x), x, nbins, out))
        return out[0::2] + 1j * out[1::2]

    def sht_forward(self, kind, nlat, nlon, lmax, mmax, x, path=None):
        """path None: serial for Gaussian, dist 1x1 for equiangular (SURVEY finding 2)."""
        if path is None:
            path = 0 if kind == GAUSSIAN else 1
        x = _c64(x).reshape(-1, nlat, nlon)
        out = np.zeros((x.shape[0], lmax, mmax, 2))
        self._check(self.L.ref_sht_forward(kind, nlat, nlon, lmax, mmax, x.shape[0], x, out,
                                           path))
        return out[..., 0] + 1j * out[..., 1]

    def sht_inverse(self, kind, nlat, nlon, coeffs):
        coeffs = np.asarray(coeffs)
        ch, lmax, mmax = coeffs.shape
        cf = np.ascontiguousarray(np.stack([coeffs.real, coeffs.imag], -1), dtype=np.float64)
        out = np.zeros((ch, nlat, nlon))
        self._check(self.L.ref_sht_inverse(kind, nlat, nlon, lmax, mmax, ch, cf, out))
        return out

    def disco_rows(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, cutoff,
                   basis=0):
        rows = np.zeros(out_nlat, dtype=np.uint64)
        K = _sz()
        self._check(self.L.ref_disco_rows(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                          out_nlon, basis, cutoff, rows, C.byref(K)))
        return rows.astype(np.int64), K.value

    def disco_entries(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, cutoff,
                      basis=0):
        rows, K = self.disco_rows(in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon,
                                  cutoff, basis)
        n = int(rows.sum()) * K
        h = np.zeros(n, dtype=np.int64)
        w = np.zeros(n, dtype=np.int64)
        v = np.zeros(n)
        b = np.zeros(n)
        self._check(self.L.ref_disco_entries(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                             out_nlon, basis, cutoff, h, w, v, b))
        return rows, K, h, w, v, b

    def disco_apply(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, cutoff, x,
                    mix, basis=0):
        mix = _c64(mix)
        cout, cin, _ = mix.shape
        y = np.zeros((cout, out_nlat, out_nlon))
        self._check(self.L.ref_disco_apply(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                           out_nlon, basis, cutoff, cin, cout, _c64(x), mix, y))
        return y

    def disco_transpose_apply(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon,
                              cutoff, x, mix, basis=0):
        mix = _c64(mix)
        cout, cin, _ = mix.shape
        y = np.zeros((cin, in_nlat, in_nlon))
        self._check(self.L.ref_disco_transpose_apply(in_kind, in_nlat, in_nlon, out_kind,
                                                     out_nlat, out_nlon, basis, cutoff, cin,
                                                     cout, _c64(x), mix, y))
        return y

    def bilinear_resample(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, x,
                          in_last_pi=0):
        x = _c64(x)
        C = x.shape[0]
        y = np.zeros((C, out_nlat, out_nlon))
        self._check(self.L.ref_bilinear_resample(in_kind, in_nlat, in_nlon, in_last_pi, out_kind,
                                                 out_nlat, out_nlon, C, x, y))
        return y

    def spectral_resample(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, x):
        x = _c64(x)
        C = x.shape[0]
        y = np.zeros((C, out_nlat, out_nlon))
        self._check(self.L.ref_spectral_resample(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                                 out_nlon, C, x, y))
        return y

    def angular_psd(self, kind, nlat, nlon, x):
        x = _c64(x)
        out = np.zeros((x.shape[0], nlat))
        self._check(self.L.ref_angular_psd(kind, nlat, nlon, x.shape[0], x, out))
        return out

    def spectral_crps_loss(self, kind, nlat, nlon, ens, obs, lmax_sum, variant):
        ens, obs = _c64(ens), _c64(obs)
        E, Cc = ens.shape[:2]
        out = np.zeros(Cc)
        self._check(self.L.ref_spectral_crps_loss(kind, nlat, nlon, E, Cc, ens, obs, lmax_sum, variant, out))
        return out

    def noise_stream(self, kind, nlat, nlon, lmax, kts, seed, steps):
        kts = _c64(kts)
        Cc = kts.shape[0]
        field = np.zeros((Cc, nlat, nlon))
        coeffs = np.zeros((Cc, lmax, lmax, 2))
        self._check(self.L.ref_noise_stream(kind, nlat, nlon, lmax, Cc, kts, seed, steps, field, coeffs))
        return field, coeffs

    def write_sfd(self, path, kind, x):
        x = _c64(x)
        self._check(self.L.ref_write_sfd(str(path).encode(), kind, x.shape[1], x.shape[2], x.shape[0], x))

    def write_weights(self, path, w1, b1):
        w1, b1 = _c64(w1), _c64(b1)
        self._check(self.L.ref_write_weights(str(path).encode(), w1.shape[0], w1.shape[1], w1, b1))

    def read_sfd(self, path, cap=1 << 22):
        """-> (code, array or None); code 0 ok, else 1 + sphere::IoErrorCode."""
        buf = np.zeros(cap)
        c, h, w = _sz(0), _sz(0), _sz(0)
        rc = self.L.ref_read_sfd(str(path).encode(), buf, cap, C.byref(c), C.byref(h), C.byref(w))
        if rc:
            return rc, None
        return 0, buf[: c.value * h.value * w.value].reshape(c.value, h.value, w.value)

    def crps_field(self, kind, nlat, nlon, ens, obs, variant):
        ens, obs = _c64(ens), _c64(obs)
        E, Cc = ens.shape[:2]
        out = np.zeros(Cc)
        self._check(self.L.ref_crps_field(kind, nlat, nlon, E, Cc, ens, obs, variant, out))
        return out

    def spectral_conv(self, kind, nlat, nlon, kernel, x):
        kernel = _c64(kernel)
        cout, cin, klmax = kernel.shape
        y = np.zeros((cout, nlat, nlon))
        self._check(self.L.ref_spectral_conv(kind, nlat, nlon, cin, cout, klmax, kernel,
                                             _c64(x), y))
        return y

    def block_apply(self, nlat, nlon, levels, embed_group, hidden, glob, cutoff, klmax, x, cond,
                    conv_w, w1, b1, w2, b2, scales):
        Cs = self.L.ref_block_channels(levels, embed_group)
        y = np.zeros((Cs, nlat, nlon))
        self._check(self.L.ref_block_apply(nlat, nlon, levels, embed_group, hidden, int(glob),
                                           cutoff, klmax, _c64(x), _c64(cond), _c64(conv_w),
                                           _c64(w1), _c64(b1), _c64(w2), _c64(b2),
                                           _c64(scales), y))
        return y

    def dist_sht_forward(self, kind, nlat, nlon, lmax, mmax, x, nh, nw):
        x = _c64(x).reshape(-1, nlat, nlon)
        out = np.zeros((x.shape[0], lmax, mmax, 2))
        csv = C.create_string_buffer(1 << 16)
        self._check(self.L.ref_dist_sht_forward(kind, nlat, nlon, lmax, mmax, x.shape[0], nh, nw,
                                                x, out, csv, 1 << 16))
        return out[..., 0] + 1j * out[..., 1], csv.value.decode()

    def dist_disco_apply(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, cutoff,
                         x, mix, nh, nw, basis=0):
        mix = _c64(mix)
        cout, cin, _ = mix.shape
        y = np.zeros((cout, out_nlat, out_nlon))
        csv = C.create_string_buffer(1 << 16)
        self._check(self.L.ref_dist_disco_apply(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                                out_nlon, basis, cutoff, cin, cout, nh, nw,
                                                _c64(x), mix, y, csv, 1 << 16))
        return y, csv.value.decode()

    def bench_sht_roundtrip(self, kind, nlat, nlon, lmax, mmax, x, nthreads, want_y=False):
        x = _c64(x).reshape(-1, nlat, nlon)
        y = np.zeros_like(x) if want_y else None
        st, tb = C.c_double(), C.c_double()
        self._check(self.L.ref_bench_sht_roundtrip(kind, nlat, nlon, lmax, mmax, x.shape[0],
                                                   nthreads, x,
                                                   None if y is None else y.ctypes.data,
                                                   C.byref(st), C.byref(tb)))
        return st.value, tb.value, y

    def bench_disco(self, in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, cutoff, x,
                    mix, nthreads, want_y=False, basis=0):
        mix = _c64(mix)
        cout, cin, _ = mix.shape
        y = np.zeros((cout, out_nlat, out_nlon)) if want_y else None
        st, asm = C.c_double(), C.c_double()
        self._check(self.L.ref_bench_disco(in_kind, in_nlat, in_nlon, out_kind, out_nlat,
                                           out_nlon, basis, cutoff, cin, cout, nthreads,
                                           _c64(x), mix, None if y is None else y.ctypes.data,
                                           C.byref(st), C.byref(asm)))
        return st.value, asm.value, y


_orc = None
_ref = None


def orc() -> _Orc:
    global _orc
    if _orc is None:
        _orc = _Orc()
    return _orc


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def random_field(shape, seed):
    """oracle::random_field (proj/tests/oracles.hpp:105-112) stream, via the C restatement."""
    return orc().random_uniform(shape, seed)
