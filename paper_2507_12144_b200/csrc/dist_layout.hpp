// Host-side layout logic of the domain-decomposed SHT and DISCO (no CUDA, no NCCL):
// which rank owns which latitude/longitude, degree/order and channel ranges, what every
// rank sends to every other rank, and the box copies that pack / unpack those payloads.
//
// Reference: the rank cube and canonical splits of distsim.hpp:45-110 (CommGrid,
// canonical_split, split_offset) and the data movement of Algorithms 1-2
// (distsim.hpp:404-547).  The reference simulator performs Alg. 1 as four per-axis
// all-to-alls (T1 W->C, T2 C->m over azimuth, T3 H->C, T4 C->l over polar); over NVSwitch
// every GPU reaches every peer at full bandwidth, so the B200 build does the pencil
// transpose of both axes in ONE all-to-all of the (polar x azimuth) plane per direction:
//
//   forward   x[C][h in H_i][w in W_j]  --A-->  x[c in C_q][H][W]  (rank q's channel slice,
//             all latitudes and longitudes) --local fused SHT--> coefficients of C_q
//             --B-->  coeffs[C][l in L_i][m in M_j]
//   inverse   the mirror image (B^-1, local inverse SHT, A^-1).
//
// Each rank's remote bytes per direction are (1 - 1/P) of its share instead of the
// reference's (1 - 1/nw) + (1 - 1/nh), coefficient payloads carry only the stored
// triangle m <= l (the reference moves the dense [lmax][mmax] block with its zeros), and
// every payload block is a contiguous run of the sender's or receiver's buffer, so the
// forward input and the inverse output need no pack / unpack pass at all.
//
// Everything here is exported through the C ABI (sph_dist_describe_*) so the CPU test
// suite executes the same schedules over gloo with numpy and the fp64 oracle.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sph {

inline std::vector<int64_t> canonical_split(int64_t n, int64_t p) {  // distsim.hpp:100-104
    std::vector<int64_t> parts(static_cast<size_t>(p), n / p);
    for (int64_t k = 0; k < n % p; ++k) ++parts[static_cast<size_t>(k)];
    return parts;
}
inline int64_t split_offset(const std::vector<int64_t>& parts, int64_t k) {  // :106-110
    int64_t off = 0;
    for (int64_t i = 0; i < k; ++i) off += parts[static_cast<size_t>(i)];
    return off;
}

// (batch, ensemble, polar, azimuth) rank cube, azimuth fastest (distsim.hpp:45-98)
struct CommGridSpec {
    std::array<int64_t, 4> sizes{1, 1, 1, 1};
    int64_t world() const { return sizes[0] * sizes[1] * sizes[2] * sizes[3]; }
    std::array<int64_t, 4> coords(int64_t rank) const {
        std::array<int64_t, 4> c{};
        c[3] = rank % sizes[3];
        rank /= sizes[3];
        c[2] = rank % sizes[2];
        rank /= sizes[2];
        c[1] = rank % sizes[1];
        c[0] = rank / sizes[1];
        return c;
    }
    int64_t rank_of(const std::array<int64_t, 4>& c) const {
        return ((c[0] * sizes[1] + c[1]) * sizes[2] + c[2]) * sizes[3] + c[3];
    }
};

// One strided 3-D block copy: n0 x n1 rows of n2 contiguous floats.
//   dst[dst_off + a*d0 + b*d1 + k] = src[src_off + a*s0 + b*s1 + k]
struct Box {
    int64_t src_off, dst_off, n0, n1, n2, s0, s1, d0, d1;
};
inline int64_t box_floats(const std::vector<Box>& bs) {
    int64_t n = 0;
    for (const auto& b : bs) n += b.n0 * b.n1 * b.n2;
    return n;
}

// all-to-all schedule in floats, indexed by plane rank
struct Exchange {
    std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_off;
    explicit Exchange(int64_t P = 0)
        : send_cnt(P, 0), send_off(P, 0), recv_cnt(P, 0), recv_off(P, 0) {}
    int64_t send_total() const { return send_off.empty() ? 0 : send_off.back() + send_cnt.back(); }
    int64_t recv_total() const { return recv_off.empty() ? 0 : recv_off.back() + recv_cnt.back(); }
    int64_t remote_send(int64_t me) const {
        int64_t n = 0;
        for (size_t p = 0; p < send_cnt.size(); ++p)
            if (static_cast<int64_t>(p) != me) n += send_cnt[p];
        return n;
    }
};

// ------------------------------------------------------------------ SHT pencil layout
// Plane rank q = i*nw + j holds latitudes H_i x longitudes W_j of the fields and degrees
// L_i x orders M_j of the coefficients (the reference's unshard layout: dim 1 over polar,
// dim 2 over azimuth, canonical splits), and computes the local SHT of channels C_q
// (canonical split of C over the P plane ranks, in plane-rank order).
//
// Coefficient payload of block (i, j) -- L_i = [l0, l1), M_j = [m0, m1) -- per channel:
// for l = l0 .. l1-1 the orders m = m0 .. min(m1, l+1)-1 as (re, im) pairs, i.e. only the
// stored triangle m <= l (harmonics.hpp:147-154 writes nothing above it).  rowoff(i,j)[k]
// is the complex offset of row l0 + k; tri(i,j) = rowoff[l1-l0] complex entries.
struct ShtLayout {
    int64_t nh = 1, nw = 1, P = 1;
    int64_t nlat = 0, nlon = 0, lmax = 0, mmax = 0, C = 0;
    std::vector<int64_t> hp, wp, lp, mp, cp;

    ShtLayout() = default;
    ShtLayout(int64_t nh_, int64_t nw_, int64_t nlat_, int64_t nlon_, int64_t lmax_, int64_t mmax_, int64_t C_)
        : nh(nh_), nw(nw_), P(nh_ * nw_), nlat(nlat_), nlon(nlon_), lmax(lmax_), mmax(mmax_), C(C_) {
        if (nh < 1 || nw < 1) throw std::invalid_argument("CommGrid: sizes must be >= 1");
        if (C < 0) throw std::invalid_argument("dist_sht: negative channel count");
        if (nlon < 2 * mmax || nlat < lmax)
            throw std::invalid_argument("dist_sht_forward: resolution insufficient for lmax/mmax");
        hp = canonical_split(nlat, nh);
        wp = canonical_split(nlon, nw);
        lp = canonical_split(lmax, nh);
        mp = canonical_split(mmax, nw);
        cp = canonical_split(C, P);
        if (hp.back() == 0 || wp.back() == 0 || lp.back() == 0 || mp.back() == 0)
            throw std::invalid_argument("shard: extent smaller than rank count");
    }
    int64_t pi(int64_t q) const { return q / nw; }
    int64_t pj(int64_t q) const { return q % nw; }
    int64_t h0(int64_t i) const { return split_offset(hp, i); }
    int64_t w0(int64_t j) const { return split_offset(wp, j); }
    int64_t l0(int64_t i) const { return split_offset(lp, i); }
    int64_t m0(int64_t j) const { return split_offset(mp, j); }
    int64_t c0(int64_t q) const { return split_offset(cp, q); }
    int64_t cq(int64_t q) const { return cp[static_cast<size_t>(q)]; }
    int64_t field_block(int64_t q) const { return hp[pi(q)] * wp[pj(q)]; }  // floats per channel
    int64_t coeff_block(int64_t q) const { return lp[pi(q)] * mp[pj(q)] * 2; }

    std::vector<int64_t> rowoff(int64_t q) const {
        const int64_t a = l0(pi(q)), n = lp[pi(q)], mb = m0(pj(q)), me = mb + mp[pj(q)];
        std::vector<int64_t> r(static_cast<size_t>(n + 1), 0);
        for (int64_t k = 0; k < n; ++k) r[k + 1] = r[k] + std::max<int64_t>(0, std::min(me, a + k + 1) - mb);
        return r;
    }
    int64_t tri(int64_t q) const { return rowoff(q).back(); }  // complex entries per channel

    // forward A: q sends channel slice C_p of its x block to p (a contiguous run of x),
    // receives [C_q][h_s][w_s] from every s
    Exchange fwd_fields(int64_t q) const {
        Exchange x(P);
        for (int64_t p = 0; p < P; ++p) {
            x.send_cnt[p] = cq(p) * field_block(q);
            x.send_off[p] = c0(p) * field_block(q);
            x.recv_cnt[p] = cq(q) * field_block(p);
            x.recv_off[p] = p ? x.recv_off[p - 1] + x.recv_cnt[p - 1] : 0;
        }
        return x;
    }
    // forward B: q sends the triangle of block p of its C_q channels, receives [C_s][tri(q)]
    // from every s -- which is [C][tri(q)] in channel order
    Exchange fwd_coeffs(int64_t q) const {
        Exchange x(P);
        for (int64_t p = 0; p < P; ++p) {
            x.send_cnt[p] = cq(q) * 2 * tri(p);
            x.send_off[p] = p ? x.send_off[p - 1] + x.send_cnt[p - 1] : 0;
            x.recv_cnt[p] = cq(p) * 2 * tri(q);
            x.recv_off[p] = c0(p) * 2 * tri(q);
        }
        return x;
    }
    // inverse A^-1 (mirror of fwd_coeffs): q sends [C_p][tri(q)] to p (channel order), receives
    // [C_q][tri(s)] from every s
    Exchange inv_coeffs(int64_t q) const {
        Exchange x(P);
        for (int64_t p = 0; p < P; ++p) {
            x.send_cnt[p] = cq(p) * 2 * tri(q);
            x.send_off[p] = c0(p) * 2 * tri(q);
            x.recv_cnt[p] = cq(q) * 2 * tri(p);
            x.recv_off[p] = p ? x.recv_off[p - 1] + x.recv_cnt[p - 1] : 0;
        }
        return x;
    }
    // inverse B^-1 (mirror of fwd_fields): q sends [C_q][h_p][w_p] blocks of its synthesized
    // fields to every p, receives channel slice C_s straight into its output block
    Exchange inv_fields(int64_t q) const {
        Exchange x(P);
        for (int64_t p = 0; p < P; ++p) {
            x.send_cnt[p] = cq(q) * field_block(p);
            x.send_off[p] = p ? x.send_off[p - 1] + x.send_cnt[p - 1] : 0;
            x.recv_cnt[p] = cq(p) * field_block(q);
            x.recv_off[p] = c0(p) * field_block(q);
        }
        return x;
    }
    // forward A unpack: recv [C_q][h_s][w_s] blocks -> full fields [C_q][nlat][nlon]
    std::vector<Box> fwd_unpack(int64_t q) const {
        const Exchange x = fwd_fields(q);
        std::vector<Box> bs;
        for (int64_t s = 0; s < P; ++s) {
            const int64_t i = pi(s), j = pj(s);
            if (cq(q) == 0) continue;
            bs.push_back({x.recv_off[s], h0(i) * nlon + w0(j), cq(q), hp[i], wp[j], hp[i] * wp[j], wp[j],
                          nlat * nlon, nlon});
        }
        return bs;
    }
    // inverse B^-1 pack: full fields [C_q][nlat][nlon] -> send blocks [C_q][h_p][w_p]
    std::vector<Box> inv_pack(int64_t q) const {
        const Exchange x = inv_fields(q);
        std::vector<Box> bs;
        for (int64_t p = 0; p < P; ++p) {
            const int64_t i = pi(p), j = pj(p);
            if (cq(q) == 0) continue;
            bs.push_back({h0(i) * nlon + w0(j), x.send_off[p], cq(q), hp[i], wp[j], nlat * nlon, nlon,
                          hp[i] * wp[j], wp[j]});
        }
        return bs;
    }
};

// ----------------------------------------------------------------- DISCO latitude layout
// Alg. 2 (distsim.hpp:468-547) reorganised around a latitude HALO.  Plane rank q = (i, j)
// holds x[C_in][H_i][W_j] (input grid) and y[C_out][Ho_i][Wo_j] (output grid).  It
// computes the output rows Ho_i for the input-channel slice Cz_j (canonical split of C_in
// over azimuth) from the input rows band(i) = the filter support of Ho_i: one all-to-all
// brings every (channel slice, halo rows, full rings) block in, then the partial sums over
// the channel slices are reduce-scattered over azimuth onto Wo_j.  This replaces the
// reference's reduce-scatter of the K-expanded partial sums over polar (2.4-4.2 GB per
// rank at 721x1440, 512 channels) with a few halo rows.
struct DiscoLayout {
    int64_t nh = 1, nw = 1, P = 1;
    int64_t hin = 0, win = 0, hout = 0, wout = 0, cin = 0, cout = 0;
    std::vector<int64_t> hp, wp, hop, wop, czp;
    std::vector<int64_t> need0, needn;  // input rows needed by polar index i

    DiscoLayout() = default;
    // band_rows(ho0, nout, &lo, &n): the input row range covering those output rows' support
    template <class BandFn>
    DiscoLayout(int64_t nh_, int64_t nw_, int64_t hin_, int64_t win_, int64_t hout_, int64_t wout_, int64_t cin_,
                int64_t cout_, BandFn band_rows)
        : nh(nh_), nw(nw_), P(nh_ * nw_), hin(hin_), win(win_), hout(hout_), wout(wout_), cin(cin_), cout(cout_) {
        if (nh < 1 || nw < 1) throw std::invalid_argument("CommGrid: sizes must be >= 1");
        hp = canonical_split(hin, nh);
        wp = canonical_split(win, nw);
        hop = canonical_split(hout, nh);
        wop = canonical_split(wout, nw);
        czp = canonical_split(cin, nw);
        if (hp.back() == 0 || wp.back() == 0 || hop.back() == 0 || wop.back() == 0)
            throw std::invalid_argument("shard: extent smaller than rank count");
        need0.resize(nh);
        needn.resize(nh);
        for (int64_t i = 0; i < nh; ++i) band_rows(split_offset(hop, i), hop[i], &need0[i], &needn[i]);
    }
    int64_t pi(int64_t q) const { return q / nw; }
    int64_t pj(int64_t q) const { return q % nw; }
    int64_t h0(int64_t i) const { return split_offset(hp, i); }
    int64_t w0(int64_t j) const { return split_offset(wp, j); }
    int64_t cz0(int64_t j) const { return split_offset(czp, j); }
    // rows of input shard i_s that polar index i needs: [r0, r0+n)
    void inter(int64_t is, int64_t i, int64_t* r0, int64_t* n) const {
        const int64_t a = std::max(h0(is), need0[i]), b = std::min(h0(is) + hp[is], need0[i] + needn[i]);
        *r0 = a;
        *n = std::max<int64_t>(0, b - a);
    }
    // A: s sends [Cz_j(p)][rows of s needed by p][W_s] to p; p receives into rows [C][need][win]
    Exchange halo(int64_t q) const {
        Exchange x(P);
        for (int64_t p = 0; p < P; ++p) {
            int64_t r0, n;
            inter(pi(q), pi(p), &r0, &n);
            x.send_cnt[p] = czp[pj(p)] * n * wp[pj(q)];
            x.send_off[p] = p ? x.send_off[p - 1] + x.send_cnt[p - 1] : 0;
            inter(pi(p), pi(q), &r0, &n);
            x.recv_cnt[p] = czp[pj(q)] * n * wp[pj(p)];
            x.recv_off[p] = p ? x.recv_off[p - 1] + x.recv_cnt[p - 1] : 0;
        }
        return x;
    }
    std::vector<Box> halo_pack(int64_t q) const {  // x[C_in][H_i][W_j] -> send
        const Exchange x = halo(q);
        const int64_t i = pi(q), j = pj(q);
        std::vector<Box> bs;
        for (int64_t p = 0; p < P; ++p) {
            int64_t r0, n;
            inter(i, pi(p), &r0, &n);
            const int64_t nc = czp[pj(p)];
            if (n == 0 || nc == 0) continue;
            bs.push_back({(cz0(pj(p)) * hp[i] + (r0 - h0(i))) * wp[j], x.send_off[p], nc, n, wp[j], hp[i] * wp[j],
                          wp[j], n * wp[j], wp[j]});
        }
        return bs;
    }
    std::vector<Box> halo_unpack(int64_t q) const {  // recv -> rows[Cz_j][need_i][win]
        const Exchange x = halo(q);
        const int64_t i = pi(q), j = pj(q);
        std::vector<Box> bs;
        for (int64_t s = 0; s < P; ++s) {
            int64_t r0, n;
            inter(pi(s), i, &r0, &n);
            const int64_t js = pj(s);
            if (n == 0 || czp[j] == 0) continue;
            bs.push_back({x.recv_off[s], (r0 - need0[i]) * win + w0(js), czp[j], n, wp[js], n * wp[js], wp[js],
                          needn[i] * win, win});
        }
        return bs;
    }
    // reduce-scatter over azimuth: partial [C_out][Ho_i][wout] -> [nw][C_out][Ho_i][mx] slots
    int64_t rs_width() const { return *std::max_element(wop.begin(), wop.end()); }
    std::vector<Box> rs_pack(int64_t q) const {
        const int64_t i = pi(q), mx = rs_width();
        std::vector<Box> bs;
        for (int64_t j = 0; j < nw; ++j)
            bs.push_back({split_offset(wop, j), j * cout * hop[i] * mx, cout, hop[i], wop[j], hop[i] * wout, wout,
                          hop[i] * mx, mx});
        return bs;
    }
    std::vector<Box> rs_unpack(int64_t q) const {
        const int64_t i = pi(q), j = pj(q), mx = rs_width();
        return {{0, 0, cout, hop[i], wop[j], hop[i] * mx, mx, hop[i] * wop[j], wop[j]}};
    }
};

}  // namespace sph
