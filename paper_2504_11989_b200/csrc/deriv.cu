// General-order derivatives of the Epstein zeta at arbitrary k (the
// polynomial-weighted zeta M^alpha(k) = sum'_z z^alpha |z|^-nu e^{-2 pi i k.z}
// = d^alpha Z(k) / (-2 pi i)^|alpha|, i.e. order-l derivative tables at k != 0).
//
// The reference only builds them at k = 0 (RegZetaTaylor, L/epstein.py:328-415), with the
// direct sum weighted by z^alpha and the reciprocal sum expanded in Hermite polynomials of the
// Gaussian (L/epstein.py:383-402).  At k != 0 the same split differentiates term by term:
//
//   d^alpha Z = pref [ 2 (2 pi)^m sum_z w_z z^alpha cos(2 pi k.z + m pi / 2)
//                      + rfac sum_{all q} d^alpha F(|k + q|^2) ],    m = |alpha| >= 1,
//   d^alpha F(|y|^2) = sum_{j_a <= alpha_a / 2} prod_a alpha_a! / (j_a! (alpha_a - 2 j_a)!)
//                       (2 y_a)^{alpha_a - 2 j_a}  F^{(m - sum j)}(|y|^2),
//   F^{(j)}(rho) = (-1)^j c^{s+j} E_{1-s-j}(c rho),
//
// where the q = 0 term is the unsplit F at y = k (it carries the singular part, so k must avoid
// the reciprocal lattice).  F^{(j)} for j in [ceil(m/2), m] come from the plan's piecewise
// tables; the q = 0 term is evaluated with E_p directly.  One thread per k point; the plan lives
// in global memory (read through L1): this path serves the derivative API, not the bench grid.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lz_internal.h"
#include "special.cuh"

namespace lz {

namespace {

// Compile-time list of the multi-indices |alpha| = M in the reference's order
// (L/epstein.py:426-433: head ascending) and of their Hermite terms.
template <int D, int M> struct DerivSpec {
    __host__ __device__ static constexpr int binom(int n, int k) {
        int r = 1;
        for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
        return r;
    }
    static constexpr int NA = binom(M + D - 1, D - 1);
    static constexpr int J0 = (M + 1) / 2;   // smallest F derivative order in the expansion
    static constexpr int NF = M - J0 + 1;    // tabulated functions F^{(J0..M)}
    static constexpr int MAXT = 64;
    struct Table {
        int alpha[NA][D];
        int n_terms;
        int t_alpha[MAXT];
        int t_exp[MAXT][D];
        int t_f[MAXT];
        double t_coef[MAXT];
    };
    __host__ __device__ static constexpr Table make() {
        Table t{};
        // enumerate alpha with |alpha| = M, head ascending (recursive order, iteratively)
        int idx = 0;
        int cur[D] = {};
        // all D-tuples with sum M in head-ascending order: count in base M + 1, digit 0 leading
        int total = 1;
        for (int a = 0; a < D; ++a) total *= (M + 1);
        for (int c = 0; c < total; ++c) {
            int rem = c, sum = 0;
            for (int a = D - 1; a >= 0; --a) {
                cur[a] = rem % (M + 1);
                rem /= (M + 1);
                sum += cur[a];
            }
            if (sum != M) continue;
            for (int a = 0; a < D; ++a) t.alpha[idx][a] = cur[a];
            ++idx;
        }
        // Hermite terms of every alpha
        int nt = 0;
        for (int i = 0; i < NA; ++i) {
            int jmax[D] = {};
            int cnt = 1;
            for (int a = 0; a < D; ++a) {
                jmax[a] = t.alpha[i][a] / 2;
                cnt *= jmax[a] + 1;
            }
            for (int c = 0; c < cnt; ++c) {
                int rem = c, jsum = 0;
                int j[D] = {};
                for (int a = 0; a < D; ++a) {
                    j[a] = rem % (jmax[a] + 1);
                    rem /= (jmax[a] + 1);
                    jsum += j[a];
                }
                double coef = 1.0;
                for (int a = 0; a < D; ++a) {
                    // alpha_a! / (j_a! (alpha_a - 2 j_a)!)
                    double f = 1.0;
                    for (int v = 2; v <= t.alpha[i][a]; ++v) f *= v;
                    for (int v = 2; v <= j[a]; ++v) f /= v;
                    for (int v = 2; v <= t.alpha[i][a] - 2 * j[a]; ++v) f /= v;
                    coef *= f;
                }
                t.t_alpha[nt] = i;
                for (int a = 0; a < D; ++a) t.t_exp[nt][a] = t.alpha[i][a] - 2 * j[a];
                t.t_f[nt] = M - jsum - J0;
                t.t_coef[nt] = coef;
                ++nt;
            }
        }
        t.n_terms = nt;
        return t;
    }
};

__device__ __forceinline__ void sincos2pi_d(double x, double& s, double& c) { sincospi(2.0 * x, &s, &c); }

template <int D, int M>
__device__ __forceinline__ void add_terms(const double (&y)[D], const double* f, double (&acc)[DerivSpec<D, M>::NA]) {
    using S = DerivSpec<D, M>;
    constexpr typename S::Table T = S::make();  // compile-time term list
    double pw[D][M + 1];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        pw[a][0] = 1.0;
#pragma unroll
        for (int e = 1; e <= M; ++e) pw[a][e] = pw[a][e - 1] * (2.0 * y[a]);
    }
#pragma unroll
    for (int t = 0; t < T.n_terms; ++t) {
        double v = T.t_coef[t] * f[T.t_f[t]];
#pragma unroll
        for (int a = 0; a < D; ++a) v *= pw[a][T.t_exp[t][a]];
        acc[T.t_alpha[t]] += v;
    }
}

// F^{(j)}(rho) from the tables (x >= x_lo), else directly
template <int NF>
__device__ __forceinline__ void fderiv(const DevDeriv& P, double rho, double (&f)[NF]) {
    const DevTable& T = P.tab;
    const double xb = fma(rho, T.r_scale, -T.x_off);
    if (xb >= T.nbins_d) {
#pragma unroll
        for (int j = 0; j < NF; ++j) f[j] = 0.0;
        return;
    }
    int e = kDirectMarker;
    double tb = 0.0;
    if (xb >= 0.0) {
        tb = (xb - 0.5) + 6755399441055744.0;
        e = __ldg(T.dir + __double2loint(tb));
    }
    if ((e & 15) == kDirectMarker) {
        const double x = rho * T.c;
#pragma unroll
        for (int j = 0; j < NF; ++j) f[j] = T.scale[j] * expint<double>(T.p[j], x);
        return;
    }
    const int L = e & 15;
    const bool lo = (e >> 4) & 1;
    const double two_l = __hiloint2double((1023 + L) << 20, 0);
    const double a = fma(xb - (tb - 6755399441055744.0), two_l, -0.5);
    const double ts = a + 6755399441055744.0;
    const int sub = __double2loint(ts);
    const TauPowers tp = tau_powers(a - (ts - 6755399441055744.0));
    if (lo) {
        const double* c = T.coef + size_t(e >> 5) + size_t(sub) * piece_stride_lo(NF);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const double cc[5] = {__ldg(c + j * kDegLo), __ldg(c + j * kDegLo + 1), __ldg(c + j * kDegLo + 2),
                                  __ldg(c + j * kDegLo + 3), __ldg(c + NF * kDegLo + j)};
            f[j] = estrin_lo(cc, tp);
        }
    } else {
        const double* c = T.coef + size_t(e >> 5) + size_t(sub) * piece_stride(NF);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            double cc[9];
#pragma unroll
            for (int m = 0; m < 8; ++m) cc[m] = __ldg(c + j * 8 + m);
            cc[8] = kDeg == 8 ? __ldg(c + NF * 8 + j) : 0.0;
            f[j] = estrin(cc, tp);
        }
    }
}

template <int D, int M>
__global__ void __launch_bounds__(128) deriv_kernel(DevDeriv P, const double* __restrict__ kin, int64_t n,
                                                    double* __restrict__ out, int* status) {
    using S = DerivSpec<D, M>;
    constexpr int NA = S::NA;
    constexpr int NF = S::NF;
    for (int64_t pt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pt < n; pt += int64_t(gridDim.x) * blockDim.x) {
        double k[D], kap[D];
#pragma unroll
        for (int a = 0; a < D; ++a) k[a] = kin[pt * D + a];
        // reduce into the cell (L/lattice.py:107-112): derivatives are periodic too
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < D; ++b) s = fma(P.A[b * D + a], k[b], s);
            kap[a] = s - floor(s + 0.5);
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < D; ++b) s = fma(P.B[a * D + b], kap[b], s);
            k[a] = s;
        }
        double acc[NA];
#pragma unroll
        for (int i = 0; i < NA; ++i) acc[i] = 0.0;
        // direct space: weights W = 2 (2 pi)^m w z^alpha (host, long double), trig phase m pi / 2
        for (int i = 0; i < P.n_dir; ++i) {
            double ph = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) ph = fma(kap[a], __ldg(P.dir_n + i * D + a), ph);
            double sn, cs;
            sincos2pi_d(ph, sn, cs);
            const double tr = (M % 4 == 0) ? cs : (M % 4 == 1) ? -sn : (M % 4 == 2) ? -cs : sn;
#pragma unroll
            for (int j = 0; j < NA; ++j) acc[j] = fma(__ldg(P.dir_w + size_t(i) * NA + j), tr, acc[j]);
        }
        // reciprocal space, exact culling per thread (q sorted by |q|)
        double kmag = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) kmag = fma(k[a], k[a], kmag);
        kmag = sqrt(kmag);
        double racc[NA];
#pragma unroll
        for (int i = 0; i < NA; ++i) racc[i] = 0.0;
        for (int i = 0; i < P.n_rec; ++i) {
            if (__ldg(P.rec_norm + i) > P.r_cut + kmag) break;
            double y[D], rho = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                y[a] = k[a] + __ldg(P.rec_q + i * D + a);
                rho = fma(y[a], y[a], rho);
            }
            double f[NF];
            fderiv<NF>(P, rho, f);
            add_terms<D, M>(y, f, racc);
        }
        // q = 0: the unsplit F at y = k (includes the singular part)
        double rho0 = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) rho0 = fma(k[a], k[a], rho0);
        if (rho0 < 1e-28) {
            if (status) atomicOr(status, 1);
        } else {
            double f0[NF];
            const double x0 = rho0 * P.tab.c;
#pragma unroll
            for (int j = 0; j < NF; ++j) f0[j] = P.tab.scale[j] * expint<double>(P.tab.p[j], x0);
            add_terms<D, M>(k, f0, racc);
        }
#pragma unroll
        for (int i = 0; i < NA; ++i) out[pt * NA + i] = P.pref * fma(P.rfac, racc[i], acc[i]);
    }
}

template <int D, int M>
cudaError_t launch_deriv_t(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 128;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > int64_t(sms) * 16) blocks = int64_t(sms) * 16;
    if (blocks < 1) blocks = 1;
    deriv_kernel<D, M><<<unsigned(blocks), threads, 0, st>>>(P, k, n, out, status);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Any order m <= 12, d <= 4: moment form.  With y = k + q,
//   d^alpha sum_q F(|y|^2) = sum_{j <= alpha/2} c(alpha, j) R[m - |j|][alpha - 2j],
//   R[p][e] = sum_q F^{(p)}(|y|^2) prod_a (2 y_a)^{e_a}          (|e| = 2p - m),
//   direct:  Dm[alpha] = sum_z W_z trig_m(2 pi k.z) z^alpha      (W_z = 2 (2 pi)^m w_z),
// so the q loop accumulates sum_p binom(2p - m + d - 1, d - 1) moments instead of every Hermite
// term of every alpha (d = 4, m = 12: 1036 + 455 moments against ~5,000 terms).  Items (direct
// points, then reciprocal points sorted by |q| up to r_cut + |k|, then q = 0 unsplit) run in
// chunks of kDgCh: each thread evaluates one item -- its trig factor or table functions, and
// the power ladders of z or 2y -- into shared memory, then every thread adds the chunk to its
// moments with compensated (Neumaier) sums (the Hermite expansion cancels at high order, the
// reason the reference combines it with fsum, L/epstein.py:383-386).  Chunks are dealt
// round-robin to gridDim.x splits; one split combines in the kernel, several through the plan's
// workspace (deriv_combine_kernel, fixed split order).
constexpr int kDgCh = 128;
constexpr int kDgDirPT = 4;   // direct moments per thread: <= 512 (455 at d = 4, m = 12)
constexpr int kDgRecPT = 9;   // reciprocal moments per thread: <= 1152 (1036 at d = 4, m = 12)

__device__ __forceinline__ void neu_add(double& s, double& c, double v) {
    const double t = s + v;
    c += fabs(s) >= fabs(v) ? (s - t) + v : (v - t) + s;
    s = t;
}

// F^{(J0 + j)}, j < nf, at rho (runtime nf)
__device__ __forceinline__ void fderiv_rt(const DevDeriv& P, double rho, double* f) {
    switch (P.nf) {
#define LZ_FCASE(N)                     \
    case N: {                           \
        double g[N];                    \
        fderiv<N>(P, rho, g);           \
        for (int j = 0; j < N; ++j) f[j] = g[j]; \
        break;                          \
    }
        LZ_FCASE(1) LZ_FCASE(2) LZ_FCASE(3) LZ_FCASE(4) LZ_FCASE(5) LZ_FCASE(6) LZ_FCASE(7)
#undef LZ_FCASE
        default: break;
    }
}

// One point's moments (hi, lo pairs in msm) -> the n_alpha outputs.
__device__ __forceinline__ void combine_point(const DevDeriv& P, const double* msm, double* orow) {
    for (int ia = threadIdx.x; ia < P.n_alpha; ia += blockDim.x) {
        double s = 0.0, c = 0.0;
        neu_add(s, c, msm[2 * ia]);
        neu_add(s, c, msm[2 * ia + 1]);
        for (int t = __ldg(P.hoff + ia); t < __ldg(P.hoff + ia + 1); ++t) {
            const int mi = P.n_dmom + __ldg(P.hmom + t);
            const double cf = P.rfac * __ldg(P.hcoef + t);
            neu_add(s, c, cf * msm[2 * mi]);
            neu_add(s, c, cf * msm[2 * mi + 1]);
        }
        if (P.add) neu_add(s, c, __ldg(P.add + ia));
        orow[ia] = P.pref * (s + c);
    }
}

template <int D>
__device__ __forceinline__ void chunk_moments(const double* sm, int rs, int cnt, unsigned long long code, double& s,
                                              double& c) {
    const int of = int(code & 0xff);
    int op[D];
#pragma unroll
    for (int a = 0; a < D; ++a) op[a] = int((code >> (8 * (a + 1))) & 0xff);
#pragma unroll 2
    for (int it = 0; it < cnt; ++it) {
        const double* r = sm + it * rs;
        double v = r[of];
#pragma unroll
        for (int a = 0; a < D; ++a) v *= r[op[a]];
        neu_add(s, c, v);
    }
}

template <int D>
__global__ void __launch_bounds__(kDgCh) deriv_moment_kernel(DevDeriv P, const double* __restrict__ kin, int64_t n,
                                                             double* __restrict__ out, int* status) {
    extern __shared__ __align__(16) double dsm[];
    const int m = P.order, nf = P.nf, rs = P.rs, tid = threadIdx.x;
    const int nsplit = gridDim.x, split = blockIdx.x;
    const int n_mom = P.n_dmom + P.n_rmom;
    double* msm = dsm + kDgCh * rs;  // [n_mom][2] (combine)
    for (int64_t pt = blockIdx.y; pt < n; pt += gridDim.y) {
        double k[D], kap[D];
        if (P.taylor) {
#pragma unroll
            for (int a = 0; a < D; ++a) k[a] = kap[a] = 0.0;
        } else {
#pragma unroll
            for (int a = 0; a < D; ++a) k[a] = kin[pt * D + a];
#pragma unroll
            for (int a = 0; a < D; ++a) {  // reduce into the cell (L/lattice.py:107-112)
                double s = 0.0;
#pragma unroll
                for (int b = 0; b < D; ++b) s = fma(P.A[b * D + a], k[b], s);
                kap[a] = s - floor(s + 0.5);
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
                double s = 0.0;
#pragma unroll
                for (int b = 0; b < D; ++b) s = fma(P.B[a * D + b], kap[b], s);
                k[a] = s;
            }
        }
        double rho0 = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) rho0 = fma(k[a], k[a], rho0);
        const double kmag = sqrt(rho0);
        // reciprocal items with |q| <= r_cut + |k| (binary search, q sorted by |q|)
        int lo = 0, hi = P.n_rec;
        const double rmax = P.r_cut + kmag;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(P.rec_norm + mid) <= rmax) lo = mid + 1;
            else hi = mid;
        }
        const int n_rq = lo, n_ritems = n_rq + (P.taylor ? 0 : 1);
        const int nd_ch = (P.n_dir + kDgCh - 1) / kDgCh, nr_ch = (n_ritems + kDgCh - 1) / kDgCh;
        double ds[kDgDirPT], dc[kDgDirPT], rsum[kDgRecPT], rc[kDgRecPT];
#pragma unroll
        for (int r = 0; r < kDgDirPT; ++r) ds[r] = dc[r] = 0.0;
#pragma unroll
        for (int r = 0; r < kDgRecPT; ++r) rsum[r] = rc[r] = 0.0;
        const int trig_case = m & 3;
        for (int ch = split; ch < nd_ch + nr_ch; ch += nsplit) {
            const bool dir = ch < nd_ch;
            const int base = (dir ? ch : ch - nd_ch) * kDgCh;
            const int cnt = min(kDgCh, (dir ? P.n_dir : n_ritems) - base);
            const int i = base + tid;
            double* rec = dsm + tid * rs;
            __syncthreads();  // the previous chunk is consumed
            if (tid < cnt) {
                double x[D];
                double f0 = 0.0;
                if (dir) {
                    double ph = 0.0;
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        ph = fma(kap[a], __ldg(P.dir_n + size_t(i) * D + a), ph);
                        x[a] = __ldg(P.dir_z + size_t(i) * D + a);
                    }
                    double sn, cs;
                    sincos2pi_d(ph, sn, cs);
                    const double tr = trig_case == 0 ? cs : trig_case == 1 ? -sn : trig_case == 2 ? -cs : sn;
                    f0 = __ldg(P.dir_w0 + i) * tr;
                    rec[0] = f0;
                } else {
                    double rho = 0.0;
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        const double y = k[a] + (i < n_rq ? __ldg(P.rec_q + size_t(i) * D + a) : 0.0);
                        x[a] = 2.0 * y;
                        rho = fma(y, y, rho);
                    }
                    double f[kMaxFunc];
                    if (i < n_rq) {
                        fderiv_rt(P, rho, f);
                    } else if (rho0 < 1e-28) {  // q = 0 at k in the reciprocal lattice: pole
                        if (status && split == 0) atomicOr(status, 1);
                        for (int j = 0; j < nf; ++j) f[j] = 0.0;
                    } else {  // q = 0, unsplit F^{(p)} (carries the singular part)
                        const double x0 = rho * P.tab.c;
                        for (int j = 0; j < nf; ++j) f[j] = P.tab.scale[j] * expint<double>(P.tab.p[j], x0);
                    }
                    for (int j = 0; j < nf; ++j) rec[j] = f[j];
                }
#pragma unroll
                for (int a = 0; a < D; ++a) {  // power ladder x_a^e, e = 0..m
                    double pw = 1.0;
                    double* pr = rec + nf + a * (m + 1);
                    for (int e = 0; e <= m; ++e) {
                        pr[e] = pw;
                        pw *= x[a];
                    }
                }
            }
            __syncthreads();
            if (dir) {
#pragma unroll
                for (int r = 0; r < kDgDirPT; ++r) {
                    const int mi = tid + r * kDgCh;
                    if (mi < P.n_dmom) chunk_moments<D>(dsm, rs, cnt, __ldg(P.mom + mi), ds[r], dc[r]);
                }
            } else {
#pragma unroll
                for (int r = 0; r < kDgRecPT; ++r) {
                    const int mi = tid + r * kDgCh;
                    if (mi < P.n_rmom) chunk_moments<D>(dsm, rs, cnt, __ldg(P.mom + P.n_dmom + mi), rsum[r], rc[r]);
                }
            }
        }
        // partial moments -> shared (one split: combine here) or the plan's workspace
        double* dst = nsplit == 1 ? msm : P.ws + (size_t(pt) * nsplit + split) * n_mom * 2;
#pragma unroll
        for (int r = 0; r < kDgDirPT; ++r) {
            const int mi = tid + r * kDgCh;
            if (mi < P.n_dmom) {
                dst[2 * mi] = ds[r];
                dst[2 * mi + 1] = dc[r];
            }
        }
#pragma unroll
        for (int r = 0; r < kDgRecPT; ++r) {
            const int mi = tid + r * kDgCh;
            if (mi < P.n_rmom) {
                dst[2 * (P.n_dmom + mi)] = rsum[r];
                dst[2 * (P.n_dmom + mi) + 1] = rc[r];
            }
        }
        if (nsplit == 1) {
            __syncthreads();
            combine_point(P, msm, out + pt * P.n_alpha);
            __syncthreads();
        }
    }
}

// Several splits per point (small batches): fixed-order sum over the splits, then the combine.
__global__ void __launch_bounds__(kDgCh) deriv_combine_kernel(DevDeriv P, int64_t n, int nsplit, double* __restrict__ out) {
    extern __shared__ __align__(16) double msm[];
    const int n_mom = P.n_dmom + P.n_rmom;
    for (int64_t pt = blockIdx.x; pt < n; pt += gridDim.x) {
        for (int mi = threadIdx.x; mi < n_mom; mi += blockDim.x) {
            double s = 0.0, c = 0.0;
            for (int sp = 0; sp < nsplit; ++sp) {
                const double* w = P.ws + ((size_t(pt) * nsplit + sp) * n_mom + mi) * 2;
                neu_add(s, c, w[0]);
                neu_add(s, c, w[1]);
            }
            msm[2 * mi] = s;
            msm[2 * mi + 1] = c;
        }
        __syncthreads();
        combine_point(P, msm, out + pt * P.n_alpha);
        __syncthreads();
    }
}

template <int D>
cudaError_t launch_deriv_g_t(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int n_mom = P.n_dmom + P.n_rmom;
    const size_t smem = sizeof(double) * (size_t(kDgCh) * P.rs + 2 * size_t(n_mom));
    cudaError_t e = cudaFuncSetAttribute(deriv_moment_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    // splits: enough CTAs for two waves when the batch is small, never more than the chunks
    const int64_t chunks = (P.n_dir + kDgCh - 1) / kDgCh + (P.n_rec + 1 + kDgCh - 1) / kDgCh;
    int64_t nsplit = 1;
    if (n < 2 * sms) nsplit = std::min<int64_t>(std::max<int64_t>(1, (2 * sms) / n), chunks);
    if (n * nsplit > kDerivWsPoints) nsplit = 1;
    // split partial moments: a stream-ordered workspace per launch (concurrent launches of one plan
    // on different streams stay independent)
    DevDeriv Q = P;
    Q.ws = nullptr;
    if (nsplit > 1) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&Q.ws), sizeof(double) * 2 * size_t(n_mom) * size_t(n * nsplit), st);
        if (e != cudaSuccess) return e;
    }
    const int64_t gy = std::min<int64_t>(n, 65535);
    deriv_moment_kernel<D><<<dim3(unsigned(nsplit), unsigned(gy)), kDgCh, smem, st>>>(Q, k, n, out, status);
    e = cudaGetLastError();
    if (e == cudaSuccess && nsplit > 1) {
        const size_t smem2 = sizeof(double) * 2 * size_t(n_mom);
        e = cudaFuncSetAttribute(deriv_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2));
        if (e == cudaSuccess) {
            deriv_combine_kernel<<<unsigned(std::min<int64_t>(n, 65535)), kDgCh, smem2, st>>>(Q, n, int(nsplit), out);
            e = cudaGetLastError();
        }
    }
    if (Q.ws) {
        const cudaError_t f = cudaFreeAsync(Q.ws, st);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

}  // namespace

int deriv_count(int d, int order) {  // binom(order + d - 1, d - 1)
    int r = 1;
    for (int i = 1; i <= d - 1; ++i) r = r * (order + i) / i;
    return r;
}

int deriv_nfunc(int order) { return order - (order + 1) / 2 + 1; }

cudaError_t launch_deriv(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
#define LZ_DCASE(DD, MM) \
    if (P.d == DD && P.order == MM) return launch_deriv_t<DD, MM>(P, k, n, out, status, st);
    LZ_DCASE(1, 1) LZ_DCASE(1, 2) LZ_DCASE(1, 3) LZ_DCASE(1, 4)
    LZ_DCASE(2, 1) LZ_DCASE(2, 2) LZ_DCASE(2, 3) LZ_DCASE(2, 4)
    LZ_DCASE(3, 1) LZ_DCASE(3, 2) LZ_DCASE(3, 3) LZ_DCASE(3, 4)
#undef LZ_DCASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_deriv_g(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    switch (P.d) {
        case 1: return launch_deriv_g_t<1>(P, k, n, out, status, st);
        case 2: return launch_deriv_g_t<2>(P, k, n, out, status, st);
        case 3: return launch_deriv_g_t<3>(P, k, n, out, status, st);
        case 4: return launch_deriv_g_t<4>(P, k, n, out, status, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lz
