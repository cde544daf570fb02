// Internal data structures shared by the host plan builder (context.cpp) and
// the sm_100a kernels (kernels.cu).  Not part of the public C ABI.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace lz {

// Branch labels of L/epstein.py:45-47.
enum Branch : int { kGeneric = 0, kLogCase = 1, kTrivial = 2 };

constexpr int kMaxDim = 4;     // L/lattice.py:20
constexpr int kMaxCtx = 4;     // distinct exponents fused into one product kernel
#ifndef LZ_LINE_PLANES
#define LZ_LINE_PLANES 24
#endif
constexpr int kLinePlanes = LZ_LINE_PLANES;  // planes per axis of the line- / row-factorised ATM direct block
constexpr int kRowRounds = 5;    // row-factorised block: most 32-item rounds of the plane sums (6 kLinePlanes <= 32 kRowRounds)
// Degree of the piecewise polynomials (kDeg + 1 coefficients): 7 or 8.  Degree 7 on bins of
// 0.125 in x saves two DFMA, one DMUL and one 16-byte load per function pair and term but needs
// ~1.8x the pieces for the same 6e-16 bound; measured slower (fcc ATM 14.4 -> 20.8 ms, C1 2^20
// 0.155 -> 0.204 ms: lanes of a warp spread over more pieces), so degree 8 is the default.
constexpr int kDeg = 8;
constexpr int kNC = kDeg + 1;
constexpr int kNCP = 10;       // per-function stride of the host fit arrays
// Device piece layout for nf functions: c0..c7 of each function (8 doubles each), then (degree 8)
// c8 of every function, padded to an even count (every double2 load 16-byte aligned).
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int piece_stride(int nf) { return kDeg == 8 ? nf * 8 + ((nf + 1) & ~1) : nf * 8; }
constexpr double kBinWidth = kDeg == 8 ? 0.25 : 0.125;  // directory bin width in x = c |y|^2
// Low-degree pieces for bins where the terms are already small (see context.cpp build_table):
// degree 4, layout c0..c3 of each function then c4 of every function (padded to even).
constexpr int kDegLo = 4;
constexpr double kLoBudget = 0.1;   // error budget of low-degree bins, in units of the cutoff
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int piece_stride_lo(int nf) { return nf * kDegLo + ((nf + 1) & ~1); }
constexpr int kDirectMarker = 15;   // directory L value meaning "evaluate E_p directly"
constexpr int kT0 = 64;             // max terms of the q = 0 power series
constexpr int kMaxFunc = 8;         // functions per table (order-12 derivatives need 7)

// ---------------------------------------------------------------------------
// Per-(lattice, nu) constants of the Crandall split (L/epstein.py:99-122, 202-259).
constexpr int kNoQuarter = -1000000;  // CtxConst::sing_q4: exponent not a multiple of 1/4
struct CtxConst {
    int branch;
    int log_m;
    int pole;            // |nu - d| < 1e-10: simple pole of the continuation at k in Lambda*
    int d;
    int sing_q4;         // 2 (nu - d) when it is an integer (|k|^{nu-d} = rho^{sing_q4/4} by square
                         // roots and products instead of pow), else kNoQuarter
    int pad_q4;
    double nu, s;        // s = s_rec = (d - nu)/2
    double pref, rfac, bconst;
    double vol, inv_vol, split, c;   // c = pi / split
    double log_t;        // log(split)
    double pi_over_t_pow_s;          // (pi/t)^s, generic t0_reg prefactor
    double sing_coef;
    double const_value;  // trivial branch value
};

// Piecewise-polynomial table of up to kMaxFunc functions f_j(x) = scale_j E_{p_j}(x),
// sharing one directory over x in [x_lo, x_hi).
struct DevTable {
    const int* dir;        // nbins entries: (first coefficient offset << 5) | lo << 4 | L ; L == 15 -> direct
    const double* coef;    // [piece][piece_stride(nfunc)], monomials in delta in [-1/2, 1/2]
    int nbins, nfunc, npieces, ncoef;   // ncoef: doubles in coef (pieces have two strides)
    double x_lo, inv_hb, x_hi;
    double c, r_scale, x_off;  // x = c rho;  bin coordinate xb = rho * r_scale - x_off
    double r_off;              // x_lo / c:  xb = (rho - r_off) * r_scale (in-cell lookup)
    double xb_max;             // largest bin coordinate evaluated (nbins - 2^-20)
    double nbins_d;            // nbins as a double (no int->FP64 conversion in the hot loop)
    double r_lo;               // |k+q| >= r_lo: low-degree bin; |k+q| < r_lo: high degree (0: no lo)
    int has_marker;            // 1 if some bin is evaluated directly (E_p; checked lookup path)
    int branchfree;            // opt-in (LATSUM_BRANCHFREE=1): select instead of the far branch
    double p[kMaxFunc], scale[kMaxFunc];  // for the direct fallback
};

// A device-resident evaluation plan: union point sets of one lattice plus the
// constants of the contexts that are evaluated together at every node.
struct DevPlan {
    int d;
    int nctx;          // contexts (plain zeta) evaluated per node
    int hess;          // 1 if context slot `hess_slot` also needs its Hessian
    int hess_slot;
    int n_dir, n_rec;
    int nw;            // direct weight channels per point (see dir_w)
    int pad_;
    double c;          // pi / split, shared by every context of the plan
    // q = 0 term as power series in rho = |k|^2 (valid for rho <= t0_rho_max, i.e. k in the BZ):
    // rows [0, nctx): t0_reg of each plain context; rows nctx, nctx+1: d/drho and d2/drho2 of
    // the Hessian context's t0_reg.  kT0 coefficients per row, n_t0 of them used.
    const double* t0c;
    int n_t0;
    int pad4_;
    double t0_rho_max;
    int alias_fp;      // 1: the Hessian's F' equals alias_ratio * (plain table 0); F' not tabulated
    int pad2_;
    double alias_ratio;
    double A[16];      // generator, row-major (columns = basis vectors)
    double B[16];      // A^{-T}, row-major
    // Direct space (one array, staged as a block): slab records [n_slabs][2d + 2] = integer
    // coordinates of (slab, first row, l0) [d], Cartesian slab center zc [d], j' of the first row,
    // (first row, row count) as two int32; row records [n_rows] = (weight row, (skip << 16) | even
    // length) as two int32; weight rows [n_dir][nw] from w_off: nctx plain channels, then (hess)
    // the Hessian weight times l'^0, l'^1, l'^2 (l' = column - slab center column).
    // device image of every staged array in the shared-memory layout (see kernels.cu stage):
    // direct block, reciprocal vectors, norms, coefficients, directory, q=0 series
    const unsigned char* blob;
    unsigned long long blob_bytes;
    const double* direct;
    const double* direct_host;  // host copy (plan-owned) for the parameter-space variant
    int n_direct, n_slabs, n_rows, rows_off, w_off, pad3_;
    double e2[4], e3[4];   // A e_{d-1}, A e_d: Cartesian row and column steps
    const double* rec_q;   // [n_rec][(d+1)&~1] Cartesian reciprocal vectors q != 0 (zero-padded), sorted by |q|
    const double* rec_norm;  // [n_rec] |q| ascending
    double r_cut;          // |k+q| > r_cut  =>  every table function is exactly zero
    double r_in;           // |k+q| <= r_in  =>  inside the table (xb < nbins, no far check)
    DevTable tab;          // functions: nctx plain F_j, then (hess) F', F''
    CtxConst ctx[kMaxCtx];
    CtxConst hctx;         // constants of the Hessian context
    // Line-factorised direct block (trace-Z ATM plans, d = 3; capi.cpp build_line_block): the
    // last section of the staged image.  At 0: v [n + 1][3] doubles (the last record zero).  Per
    // lattice axis a, at line_slot_off[a]: slot words [K][32] (uint32: byte offset of the v record
    // | 16 x step code << 16), K = line_K[a]; at
    // line_meta_off[a]: each lane's first (n_b, n_c) as int16 pairs [32], then the lane range of
    // every plane n_a = m (uint8 glo[line_P[a] + 1]).  Hessian channel weight = line_sign v v^T.
    const double* q0_host;  // host copy (plan-owned) of the Hessian q = 0 pieces [q0_nb][piece_stride(2)]
    int q0_nb, pad5_;       // (line kernel; 0: no pieces, the line kernel is not used)
    double q0_inv_h;        // bins per unit rho (c / kBinWidth)
    double h_kk;            // Hessian context: sing_coef inv_vol / (pref rfac)
    double h_cm;            // Hessian context: -4 pref rfac / (4 pi^2) (M = h_cm (Y + delta G1 / 2))
    const double* t0_host;  // host copy (plan-owned) of the q = 0 series rows [nctx + 2][kT0]
    const double* rq_host;  // host copy (plan-owned) of rec_q at the padded stride (d + 1) & ~1
    unsigned line_bytes;   // 0: no line block
    int line_K[3], line_P[3], line_slot_off[3], line_meta_off[3];
    double line_sign;
    // Row-factorised direct block (capi.cpp build_row_block; global memory, read only by
    // row_table_kernel): per axis a the half lattice {(n_a, n_b, n_c) >lex 0} grouped into rows
    // (m = n_a, j = n_b).  row_pts: 4 doubles per point (n_c, v), rows contiguous; row_idx:
    // (first point, length) of row (a, jj = j - row_jmin[a], m) at [(a row_nJ + jj) row_PS + m].
    // The table kernel writes D[a][iu][jj][item = 6 m + channel] (complex, row_NI items per row
    // index, zero where no row exists) for every radial node; line_P[a] = planes of axis a.
    const double* row_pts;
    const int* row_idx;
    int row_on;            // 1: the ATM kernel takes its plane sums from the D table
    int row_nJ, row_PS, row_NI;
    int row_jmin[3];
    int row_cand_max;      // candidate-list capacity used by the kernel (<= kRowCand; LATSUM_ROW_CAND_MAX, tests)
};

// Derivative plan (deriv.cu): one context, derivatives of total order `order` (0..12) at
// arbitrary k (or, in Taylor mode, of Z_reg at k = 0).  Plain global-memory arrays (read
// through L1).
struct DevDeriv {
    int d, order, n_dir, n_rec;
    double A[16], B[16];
    const double* dir_n;     // [n_dir][d] integer coordinates (half lattice)
    const double* dir_w;     // [n_dir][n_alpha] 2 (2 pi)^m w z^alpha (compile-time kernel)
    const double* rec_q;     // [n_rec][d] sorted by |q|
    const double* rec_norm;  // [n_rec]
    double r_cut, pref, rfac;
    DevTable tab;            // F^{(j)}, j = ceil(m/2) .. m
    // moment form (deriv.cu deriv_moment_kernel; any order <= 12, d <= 4)
    const double* dir_z;     // [n_dir][d] Cartesian z
    const double* dir_w0;    // [n_dir] 2 (2 pi)^m w_z
    const unsigned long long* mom;  // packed offsets into an item record: byte 0 = function
                                    // slot, byte 1 + a = power-ladder slot of axis a
    int n_alpha, n_dmom, n_rmom, nf;  // moments: n_dmom direct (one per alpha), then n_rmom reciprocal
    int rs;                  // doubles per item record: nf function slots + d (order + 1) powers
    int taylor;              // 1: Z_reg at k = 0 (no q = 0 item; `add` carries bconst and the
                             // q = 0 series term), 0: d^alpha Z at the given k (q = 0 unsplit)
    const int* hoff;         // [n_alpha + 1] Hermite terms of each alpha ...
    const int* hmom;         // ... their reciprocal moment index ...
    const double* hcoef;     // ... and coefficient prod_a alpha_a! / (j_a! (alpha_a - 2 j_a)!)
    const double* add;       // [n_alpha] added inside the pref bracket (Taylor mode), or null
    double* ws;              // split partial moments [points x splits][n_dmom + n_rmom][2] (per launch)
};
constexpr int kDerivWsPoints = 296;  // most (point, split) pairs of one split launch (2 x 148 SMs)

// Fixed Duffy grid description (device arrays + patch decomposition).
struct DevGrid {
    const double* u;   // radial nodes in (0, 1/2)
    const double* wu;  // radial weights incl. grading Jacobian and u^{d-1}
    const double* v;   // angular nodes on [0, 1/2]
    const double* wv;  // angular weights
    int n_u, n_v, n_cell, pu, pv, npu, npv, nv2;
    int64_t tile_lo, tile_hi, n_patch;
    double* wpart;             // [n_tiles * 8][ncomp] warp partials (scratch)
    unsigned int* tcount;      // [n_tiles] arrival counters, zero between launches
    unsigned int* work;        // [2] line kernel work queue: next ticket, warps done (zero between launches)
    double* dtab;              // row-factorised ATM kernel: D table [3][n_u][row_nJ][row_NI] complex (scratch)
};


// Host-side mirror of one context: constants + enumerated sets (host memory).
struct HostCtx {
    int d;
    double A[16], B[16];
    CtxConst k;
    double kmax;
    // plain evaluation sets (L/epstein.py:156-198)
    std::vector<double> dir_n, dir_z, dir_w;   // n (int coords), z = A n, weights
    std::vector<double> rec_n, rec_q;          // n, q = B n
    // widened sets for the Hessian (poly_order = 2, gamma order s + 2)
    int want_hess = 0;   // requested at creation (deriv_order >= 2)
    int has_hess = 0;    // sets enumerated
    int ball_sets = 0;   // plan-private context: Hessian direct set cut to the ball that matters
    std::vector<double> hdir_n, hdir_z, hdir_w;
    std::vector<double> hrec_n, hrec_q;
};

struct HostTable {
    std::vector<int> dir;
    std::vector<double> coef;
    int nbins = 0, nfunc = 0, npieces = 0;
    double x_lo = 0, inv_hb = 0, x_hi = 0;
    double p[kMaxFunc] = {}, scale[kMaxFunc] = {};
    double max_rel_err = 0;   // measured during the build (degree-kDeg pieces)
    int n_lo_bins = 0;        // bins with degree-kDegLo pieces
    int lo_start = 0;         // first low-degree bin (low-degree bins form the suffix)
};

#ifndef LZ_LO_HORNER
#define LZ_LO_HORNER 1
#endif
// Degree-kDeg polynomial in Estrin form: dependency depth 3-4 instead of 7-8, and the
// powers tau^2, tau^4 (, tau^8) are shared by every function of a table row.
// Host (table build check) and device evaluate with the same operation order.
struct TauPowers {
    double t1, t2, t4, t8;
};
#ifdef __CUDACC__
__host__ __device__
#endif
inline TauPowers tau_powers(double t) {
    TauPowers p;
    p.t1 = t;
    p.t2 = t * t;
    p.t4 = p.t2 * p.t2;
    p.t8 = p.t4 * p.t4;
    return p;
}
#ifdef __CUDACC__
__host__ __device__
#endif
inline double estrin(const double* c, const TauPowers& p) {
    const double a0 = fma(c[1], p.t1, c[0]);
    const double a1 = fma(c[3], p.t1, c[2]);
    const double a2 = fma(c[5], p.t1, c[4]);
    const double a3 = fma(c[7], p.t1, c[6]);
    const double b0 = fma(a1, p.t2, a0);
    const double b1 = fma(a3, p.t2, a2);
    const double e0 = fma(b1, p.t4, b0);
    if (kDeg == 8) return fma(c[8], p.t8, e0);
    return e0;
}
#ifdef __CUDACC__
__host__ __device__
#endif
inline double estrin_lo(const double* c, const TauPowers& p) {  // degree 4
#if LZ_LO_HORNER
    // Horner: no tau powers (2 DMUL fewer per table term; the degree-4 bins carry most terms)
    return fma(fma(fma(fma(c[4], p.t1, c[3]), p.t1, c[2]), p.t1, c[1]), p.t1, c[0]);
#else
    const double a0 = fma(c[1], p.t1, c[0]);
    const double a1 = fma(c[3], p.t1, c[2]);
    const double b0 = fma(a1, p.t2, a0);
    return fma(c[4], p.t4, b0);
#endif
}

// Errors raised by the host builder carry an lz status code.
struct Error {
    int code;
    std::string msg;
};

// context.cpp
void build_context(int d, const double* a, double nu, double splitting, int deriv_order,
                   HostCtx* out);
// term_cutoff: terms below it (relative to the unit scale |rfac pref|) end the table; 1e-18 is the
// reference's term cutoff (L/epstein.py:51)
void build_table(const double* p, const double* scale, int nfunc, double c, double x_lo,
                 double rfac_pref, HostTable* out, double poly_pow = 1.0, double term_cutoff = 1e-18);
// the fused ATM plan's term cutoff (table end and direct ball): its lattice sums are bit-identical
// at 1e-18 and 1e-16 (fcc: 19.182931071888479 both), the terms it drops are below the rounding of
// every node's FP64 Hessian (capi.cpp build_host_plan)
constexpr double kAtmTermCutoff = 1e-16;
// Point sets of the order-`order` derivative tables (L/epstein.py:376-377): direct weights
// widened by |z|^order, reciprocal Gamma order s + order, cutoff 1e-20.
void build_deriv_sets(const HostCtx& h, int order, std::vector<double>* dir_n, std::vector<double>* rec_n);
double table_x_lo(const HostCtx& h);
// Degree-kDeg Chebyshev interpolant of f on [x0, x1] as monomials in delta in [-1/2, 1/2] (the
// device's piece layout); returns the worst absolute error at 21 points (device evaluation order).
double fit_piece_fn(const std::function<long double(long double)>& f, long double x0, long double x1, double* out);
void build_hess_sets(HostCtx& h);
long double t0_coeff(const CtxConst& k, int n);   // rho-series coefficient of t0_reg
void build_reg_derivatives(const HostCtx& h, int order, std::vector<int>* alphas, std::vector<double>* vals);
void gauss_legendre(int n, std::vector<double>* x, std::vector<double>* w);  // on [-1, 1]
// body(i) for i in [0, n) on up to 32 host threads (dynamic chunks of `grain`); serial when
// n < 2 * grain.  Host setup only (table fits, plan weights).
void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t)>& body);

}  // namespace lz
