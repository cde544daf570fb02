// Host-side plan builder: lattice geometry, exponent classification, the
// truncated direct/reciprocal point sets and the Crandall constants of one
// (lattice, nu) context, plus the piecewise-polynomial tables of the radial
// reciprocal summand.  One-time setup per context; everything is computed in
// long double and rounded once.
//
// Follows, in order:
//   classify_exponent          L/epstein.py:58-70
//   _integer_shell/_lex_pos    L/epstein.py:73-90
//   EpsteinContext.__init__    L/epstein.py:99-122
//   _enumerate_direct          L/epstein.py:126-154
//   _enumerate_reciprocal      L/epstein.py:159-194
//   singular_coef              L/epstein.py:202-215
//   BrillouinZone.corner_radius L/lattice.py:131-136
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "lz_internal.h"
#include "special.cuh"

namespace lz {

using ld = long double;
static const ld kPiL = 3.141592653589793238462643383279502884L;

namespace {

constexpr double kBranchTol = 1e-12;   // L/epstein.py:49
constexpr double kPoleTol = 1e-10;     // L/epstein.py:50
constexpr double kTermCutoff = 1e-18;  // L/epstein.py:51
constexpr int kMaxShells = 80;         // L/epstein.py:52

void fail(int code, const std::string& m) { throw Error{code, m}; }

// det and inverse of a small dense matrix by Gaussian elimination (long double)
ld det_inv(int d, const ld* a, ld* inv) {
    ld m[kMaxDim][2 * kMaxDim];
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < 2 * d; ++j) m[i][j] = j < d ? a[i * d + j] : (j - d == i ? 1.0L : 0.0L);
    ld det = 1.0L;
    for (int col = 0; col < d; ++col) {
        int piv = col;
        for (int r = col + 1; r < d; ++r)
            if (std::fabs(m[r][col]) > std::fabs(m[piv][col])) piv = r;
        if (m[piv][col] == 0.0L) return 0.0L;
        if (piv != col) {
            for (int j = 0; j < 2 * d; ++j) std::swap(m[piv][j], m[col][j]);
            det = -det;
        }
        det *= m[col][col];
        ld pv = m[col][col];
        for (int j = 0; j < 2 * d; ++j) m[col][j] /= pv;
        for (int r = 0; r < d; ++r) {
            if (r == col) continue;
            ld f = m[r][col];
            if (f == 0.0L) continue;
            for (int j = 0; j < 2 * d; ++j) m[r][j] -= f * m[col][j];
        }
    }
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) inv[i * d + j] = m[i][d + j];
    return det;
}

// Integer vectors with max-norm exactly r, lexicographic (first index slowest).
std::vector<int> integer_shell(int d, int r) {
    std::vector<int> out;
    if (r == 0) {
        out.assign(d, 0);
        return out;
    }
    // lexicographic order over [-r, r]^d (first coordinate most significant), max-norm r only:
    // walk the prefixes; a prefix below r admits only the last coordinates -r and +r
    const int w = 2 * r + 1;
    long nprefix = 1;
    for (int i = 0; i < d - 1; ++i) nprefix *= w;
    std::vector<int> n(d);
    for (long idx = 0; idx < nprefix; ++idx) {
        long rem = idx;
        int mx = 0;
        for (int i = d - 2; i >= 0; --i) {
            n[i] = int(rem % w) - r;
            rem /= w;
            mx = std::max(mx, std::abs(n[i]));
        }
        if (mx == r) {
            for (int last = -r; last <= r; ++last) {
                n[d - 1] = last;
                out.insert(out.end(), n.begin(), n.end());
            }
        } else {
            n[d - 1] = -r;
            out.insert(out.end(), n.begin(), n.end());
            n[d - 1] = r;
            out.insert(out.end(), n.begin(), n.end());
        }
    }
    return out;
}

bool lex_positive(const int* n, int d) {
    for (int i = 0; i < d; ++i) {
        if (n[i] > 0) return true;
        if (n[i] < 0) return false;
    }
    return false;
}


}  // namespace

// ---------------------------------------------------------------------------
static void classify(double nu, int d, CtxConst* k) {
    if (!std::isfinite(nu)) fail(1, "exponent must be finite");
    if (std::fabs(nu) > 100.0) fail(1, "exponent magnitude above 100 is not supported");
    // Python round() is round-half-even: nearbyint under the default mode.
    double m = std::nearbyint((nu - d) / 2.0);
    if (m >= 0 && std::fabs(nu - (d + 2 * m)) < kBranchTol) {
        k->branch = kLogCase;
        k->nu = double(d + 2 * m);
        k->log_m = int(m);
        return;
    }
    double j = std::nearbyint(-nu / 2.0);
    if (j >= 0 && std::fabs(nu + 2 * j) < kBranchTol) {
        k->branch = kTrivial;
        k->nu = -2.0 * j;
        k->log_m = -1;
        return;
    }
    k->branch = kGeneric;
    k->nu = nu;
    k->log_m = -1;
}

// r2_ball > 0 (plan-private Hessian sets): points with |z|^2 > r2_ball are skipped without their
// Gamma function -- the shells' cube corners, whose terms lie below 1e-3 of the cutoff and which
// the plan's ball truncation drops anyway.
static void enumerate_direct(const HostCtx& h, int poly_order, double tol, std::vector<double>* pn,
                             std::vector<double>* pz, std::vector<double>* pw, double r2_ball = 0.0) {
    const int d = h.d;
    const ld nu = h.k.nu, t = h.k.split;
    pn->clear();
    pz->clear();
    pw->clear();
    ld total = 1.0L;
    int below = 0;
    bool done = false;
    for (int r = 1; r <= kMaxShells; ++r) {
        std::vector<int> shell = integer_shell(d, r);
        const int cnt = int(shell.size()) / d;
        std::vector<int> idx;
        for (int i = 0; i < cnt; ++i)
            if (lex_positive(&shell[i * d], d)) idx.push_back(i);
        const int m = int(idx.size());
        std::vector<double> sn(size_t(m) * d), sz(size_t(m) * d), sw(m);
        std::vector<ld> smag(m);
        std::vector<char> out(m, 0);
        // per point in parallel (large shells), reduced below in the fixed point order.  The
        // weight depends on |z|^2 only, so the shell's points are grouped by it first (sorted;
        // equal within 64 long-double roundings) and one point per group evaluates the Gamma
        // function -- a symmetric lattice has a handful of distinct radii per max-norm shell.
        std::vector<ld> r2s(m);
        parallel_for(m, 512, [&](int64_t j) {
            const int* n = &shell[idx[j] * d];
            ld r2 = 0.0L;
            for (int a = 0; a < d; ++a) {
                ld za = 0.0L;
                for (int b = 0; b < d; ++b) za += ld(h.A[a * d + b]) * n[b];
                sn[size_t(j) * d + a] = double(n[a]);
                sz[size_t(j) * d + a] = double(za);
                r2 += za * za;
            }
            r2s[j] = r2;
        });
        std::vector<int> ord(m), rep, group(m);
        for (int j = 0; j < m; ++j) ord[j] = j;
        std::sort(ord.begin(), ord.end(), [&](int a, int b) { return r2s[a] < r2s[b] || (r2s[a] == r2s[b] && a < b); });
        for (int s = 0; s < m; ++s) {
            if (s == 0 || r2s[ord[s]] - r2s[ord[rep.back()]] > 64.0L * LDBL_EPSILON * r2s[ord[s]]) rep.push_back(s);
            group[ord[s]] = int(rep.size()) - 1;
        }
        std::vector<double> gw(rep.size());
        std::vector<ld> gmag(rep.size());
        std::vector<char> gout(rep.size(), 0);
        parallel_for(int64_t(rep.size()), 16, [&](int64_t gi) {
            const ld r2 = r2s[ord[rep[gi]]];
            if (r2_ball > 0.0 && double(r2) > r2_ball) {
                gout[gi] = 1;
                gmag[gi] = 0.0L;
                gw[gi] = 0.0;
                return;
            }
            // truncation decisions and the reported weights need double precision only (the
            // reference computes them in double)
            const double xd = double(kPiL * t * r2), r2d = double(r2), nud = double(nu);
            const double w = upper_gamma<double>(nud / 2.0, xd) * std::pow(r2d, -nud / 2.0);
            gmag[gi] = std::fabs(ld(w)) * ld(std::pow(r2d, double(poly_order) / 2.0));
            gw[gi] = w;
        });
        for (int j = 0; j < m; ++j) {
            out[j] = gout[group[j]];
            smag[j] = gmag[group[j]];
            sw[j] = gw[group[j]];
        }
        ld mag = 0.0L, wsum = 0.0L;
        for (int j = 0; j < m; ++j) {
            mag = std::max(mag, smag[j]);
            wsum += std::fabs(ld(sw[j]));
        }
        if (mag > ld(tol) * total) {
            for (int j = 0; j < m; ++j) {
                if (out[j]) continue;
                pn->insert(pn->end(), sn.begin() + size_t(j) * d, sn.begin() + size_t(j + 1) * d);
                pz->insert(pz->end(), sz.begin() + size_t(j) * d, sz.begin() + size_t(j + 1) * d);
                pw->push_back(sw[j]);
            }
            total += wsum;
            below = 0;
        } else if (++below >= 2) {
            done = true;
            break;
        }
    }
    if (!done) fail(6, "direct-space sum did not truncate within shell budget");
}

static void enumerate_reciprocal(const HostCtx& h, double gamma_order, double tol,
                                 std::vector<double>* pn, std::vector<double>* pq) {
    const int d = h.d;
    const ld nu = h.k.nu, t = h.k.split, kmax = h.kmax;
    pn->clear();
    pq->clear();
    ld total = 1.0L;
    int below = 0;
    bool done = false;
    for (int r = 1; r <= kMaxShells; ++r) {
        std::vector<int> shell = integer_shell(d, r);
        const int cnt = int(shell.size()) / d;
        ld mag = 0.0L;
        bool inf = false;
        std::vector<ld> rq(cnt);
        std::vector<double> sq(size_t(cnt) * d);
        for (int i = 0; i < cnt; ++i) {
            ld r2 = 0.0L;
            for (int a = 0; a < d; ++a) {
                ld q = 0.0L;
                for (int b = 0; b < d; ++b) q += ld(h.B[a * d + b]) * shell[i * d + b];
                sq[size_t(i) * d + a] = double(q);
                r2 += q * q;
            }
            rq[i] = std::sqrt(r2);
            if (rq[i] - kmax <= 0.05L) inf = true;
        }
        if (!inf) {
            std::vector<ld> bnd(cnt);
            parallel_for(cnt, 128, [&](int64_t i) {
                ld r_low = rq[i] - kmax;
                ld x_low = kPiL * r_low * r_low / t;
                ld r_pow = (nu >= d) ? rq[i] + kmax : r_low;
                bnd[i] = std::fabs(upper_gamma<double>(gamma_order, double(x_low))) *
                         std::pow(double(r_pow), double(nu) - d);
            });
            for (int i = 0; i < cnt; ++i) mag = std::max(mag, ld(bnd[i]));
        }
        if (inf || mag > ld(tol) * total) {
            for (int i = 0; i < cnt; ++i)
                for (int a = 0; a < d; ++a) pn->push_back(double(shell[i * d + a]));
            pq->insert(pq->end(), sq.begin(), sq.end());
            if (!inf) total += mag;
            below = 0;
        } else if (++below >= 2) {
            done = true;
            break;
        }
    }
    if (!done) fail(6, "reciprocal-space sum did not truncate within shell budget");
}

void build_context(int d, const double* a, double nu, double splitting, int deriv_order,
                   HostCtx* h) {
    if (d < 1 || d > kMaxDim) fail(7, "dimension outside supported range 1..4");
    for (int i = 0; i < d * d; ++i)
        if (!std::isfinite(a[i])) fail(7, "generator contains non-finite entries");
    h->d = d;
    std::memset(h->A, 0, sizeof(h->A));
    std::memset(h->B, 0, sizeof(h->B));
    ld al[16], inv[16];
    for (int i = 0; i < d * d; ++i) {
        al[i] = a[i];
        h->A[i] = a[i];
    }
    ld det = det_inv(d, al, inv);
    if (!(std::fabs(det) >= 1e-300L) || !std::isfinite(double(det)))
        fail(7, "generator matrix is singular");
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) h->B[i * d + j] = double(inv[j * d + i]);  // A^{-T}
    CtxConst& k = h->k;
    std::memset(&k, 0, sizeof(k));
    k.d = d;
    classify(nu, d, &k);
    k.vol = double(std::fabs(det));
    k.inv_vol = 1.0 / k.vol;
    ld vol = std::fabs(det);
    ld t = splitting > 0 ? ld(splitting) : std::pow(vol, -2.0L / d);
    k.split = double(t);
    k.c = double(kPiL / t);
    k.log_t = double(std::log(t));
    k.pole = std::fabs(k.nu - d) < kPoleTol ? 1 : 0;
    // corner radius of the Brillouin zone box
    ld kmax = 0.0L;
    for (int corner = 0; corner < (1 << d); ++corner) {
        ld r2 = 0.0L;
        for (int i = 0; i < d; ++i) {
            ld v = 0.0L;
            for (int j = 0; j < d; ++j) v += ld(h->B[i * d + j]) * (((corner >> (d - 1 - j)) & 1) ? 0.5L : -0.5L);
            r2 += v * v;
        }
        kmax = std::max(kmax, std::sqrt(r2));
    }
    h->kmax = double(kmax);
    if (k.branch == kTrivial) {
        k.const_value = k.nu == 0.0 ? -1.0 : 0.0;
        return;
    }
    const ld nul = k.nu;
    k.s = double((ld(d) - nul) / 2.0L);
    k.pref = double(1.0L / std::tgamma(nul / 2.0L));
    k.rfac = double(std::pow(kPiL, nul - ld(d) / 2.0L) / vol);
    k.bconst = double(-2.0L * std::pow(kPiL * t, nul / 2.0L) / nul);
    {
        const double q4 = 2.0 * (k.nu - double(d));
        k.sing_q4 = (std::fabs(q4 - std::nearbyint(q4)) < 1e-12 && std::fabs(q4) <= 64.0) ? int(std::nearbyint(q4))
                                                                                          : kNoQuarter;
    }
    k.pi_over_t_pow_s = double(std::pow(kPiL / t, (ld(d) - nul) / 2.0L));
    if (k.branch == kLogCase) {
        int m = k.log_m;
        ld fact = 1.0L;
        for (int i = 2; i <= m; ++i) fact *= i;
        k.sing_coef = double(std::pow(kPiL, 2.0L * m + ld(d) / 2.0L) / std::tgamma(ld(m) + ld(d) / 2.0L) *
                             ((m + 1) % 2 == 0 ? 1.0L : -1.0L) / fact);
    } else {
        k.sing_coef = double(std::pow(kPiL, nul - ld(d) / 2.0L) * std::tgamma((ld(d) - nul) / 2.0L) /
                             std::tgamma(nul / 2.0L));
    }
    // deriv_order < 0: plan-private contexts (ATM plans) that need only part of the sets --
    // -1: constants and the reciprocal set; -2: constants and the Hessian sets
    h->want_hess = (deriv_order >= 2 || deriv_order == -2) ? 1 : 0;
    h->ball_sets = deriv_order == -2 ? 1 : 0;  // plan-private: skip the shells' far cube corners
    // the Hessian's widened sets (needed by every Hessian / ATM plan) are enumerated on a second
    // thread while the plain sets are: context creation costs the longer of the two
    std::future<void> hess;
    if (h->want_hess) hess = std::async(std::launch::async, [h] { build_hess_sets(*h); });
    if (deriv_order >= 0) enumerate_direct(*h, 0, kTermCutoff, &h->dir_n, &h->dir_z, &h->dir_w);
    if (deriv_order != -2) enumerate_reciprocal(*h, k.s, kTermCutoff, &h->rec_n, &h->rec_q);
    if (hess.valid()) hess.get();
}

// Plan-private Hessian direct set (ball_sets): every lex-positive lattice point with |z|^2 <=
// r2_ball, enumerated directly -- outer coordinates over their bounding ranges (|n_a| <= R |b_a|,
// b_a the a-th reciprocal basis vector), the last one from the quadratic |A n|^2 <= R^2 -- instead
// of max-norm shells whose cube corners lie far outside the ball.  Weights as in enumerate_direct
// (double precision, one Gamma function per distinct |z|^2).  The order of the points is the
// enumeration's; the plan sorts them itself.
static void enumerate_ball(const HostCtx& h, double r2_ball, std::vector<double>* pn, std::vector<double>* pz,
                           std::vector<double>* pw) {
    const int d = h.d;
    const ld R2 = ld(r2_ball), R = std::sqrt(R2);
    pn->clear();
    pz->clear();
    pw->clear();
    long lim[kMaxDim];
    for (int a = 0; a < d; ++a) {
        ld nb = 0.0L;  // |b_a|^2, b_a = a-th row of A^{-1} = a-th column of B
        for (int r = 0; r < d; ++r) nb += ld(h.B[r * d + a]) * h.B[r * d + a];
        lim[a] = long(std::floor(R * std::sqrt(nb) * (1.0L + 1e-12L))) + 1;
    }
    ld al[kMaxDim], aa = 0.0L;  // last basis vector (column d - 1 of A)
    for (int r = 0; r < d; ++r) {
        al[r] = h.A[r * d + (d - 1)];
        aa += al[r] * al[r];
    }
    std::vector<ld> r2s;
    long n[kMaxDim] = {0, 0, 0, 0};
    // odometer over the outer coordinates n_0 .. n_{d-2}
    for (int a = 0; a + 1 < d; ++a) n[a] = -lim[a];
    if (d >= 2) n[0] = 0;  // lex-positive points have n_0 >= 0
    for (;;) {
        ld zo[kMaxDim], cc = 0.0L, bb = 0.0L;
        for (int r = 0; r < d; ++r) {
            zo[r] = 0.0L;
            for (int a = 0; a + 1 < d; ++a) zo[r] += ld(h.A[r * d + a]) * n[a];
            cc += zo[r] * zo[r];
            bb += zo[r] * al[r];
        }
        const ld disc = bb * bb - aa * (cc - R2);
        if (disc >= 0.0L) {
            const ld sq = std::sqrt(disc);
            const long lo = long(std::ceil((-bb - sq) / aa - 1e-9L)), hi = long(std::floor((-bb + sq) / aa + 1e-9L));
            for (long l = lo; l <= hi; ++l) {
                n[d - 1] = l;
                int nn[kMaxDim];
                for (int a = 0; a < d; ++a) nn[a] = int(n[a]);
                if (!lex_positive(nn, d)) continue;
                ld r2 = 0.0L, z[kMaxDim];
                for (int r = 0; r < d; ++r) {
                    z[r] = zo[r] + al[r] * l;
                    r2 += z[r] * z[r];
                }
                if (r2 > R2) continue;
                for (int a = 0; a < d; ++a) {
                    pn->push_back(double(n[a]));
                    pz->push_back(double(z[a]));
                }
                r2s.push_back(r2);
            }
        }
        int a = d - 2;
        for (; a >= 0; --a) {
            if (++n[a] <= lim[a]) break;
            n[a] = a == 0 ? 0 : -lim[a];
        }
        if (a < 0) break;
    }
    // groups of equal |z|^2 as rounded to double (these weights are double-precision and serve
    // the plan's truncation decisions only; the plan recomputes the kept ones in long double)
    const size_t m = r2s.size();
    pw->assign(m, 0.0);
    std::unordered_map<uint64_t, uint32_t> seen;
    seen.reserve(m / 4 + 16);
    std::vector<uint32_t> group(m);
    std::vector<double> gr2;
    for (size_t j = 0; j < m; ++j) {
        const double r2d = double(r2s[j]);
        uint64_t bits;
        std::memcpy(&bits, &r2d, sizeof(bits));
        const auto it = seen.emplace(bits, uint32_t(gr2.size()));
        if (it.second) gr2.push_back(r2d);
        group[j] = it.first->second;
    }
    std::vector<double> gw(gr2.size());
    const double nud = h.k.nu, td = h.k.split;
    parallel_for(int64_t(gr2.size()), 16, [&](int64_t gi) {
        gw[gi] = upper_gamma<double>(nud / 2.0, double(kPiL) * td * gr2[gi]) * std::pow(gr2[gi], -nud / 2.0);
    });
    for (size_t j = 0; j < m; ++j) (*pw)[j] = gw[group[j]];
}

void build_hess_sets(HostCtx& h) {
    if (h.has_hess || !h.want_hess || h.k.branch == kTrivial) return;
    // Hessian sets: the derivative-table enumerators of L/epstein.py:376-377
    // specialised to second order (z^alpha weight |z|^2, gamma order s + 2).
    double r2_ball = 0.0;
    if (h.ball_sets) {
        // radius where w |z|^2 (w = Gamma(nu/2, pi t r2) r2^-nu/2, decreasing) falls to 1e-3 of
        // the term cutoff relative to a unit total (the plan's totals exceed one)
        const double nu = h.k.nu, t = h.k.split, target = 1e-3 * kTermCutoff;
        auto f = [&](double r2) {
            return upper_gamma<double>(nu / 2.0, double(kPiL) * t * r2) * std::pow(r2, -nu / 2.0) * std::max(1.0, r2);
        };
        double lo = 1e-3, hi = 1e-3;
        while (f(hi) > target && hi < 1e8) hi *= 2.0;
        if (hi < 1e8) {
            for (int it = 0; it < 60; ++it) {
                const double mid = 0.5 * (lo + hi);
                (f(mid) > target ? lo : hi) = mid;
            }
            r2_ball = hi * (1.0 + 1e-9);
        }
    }
    const bool tm = std::getenv("LATSUM_TIMING") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    if (r2_ball > 0.0) enumerate_ball(h, r2_ball, &h.hdir_n, &h.hdir_z, &h.hdir_w);
    else enumerate_direct(h, 2, kTermCutoff, &h.hdir_n, &h.hdir_z, &h.hdir_w, 0.0);
    auto t1 = std::chrono::steady_clock::now();
    enumerate_reciprocal(h, h.k.s + 2.0, kTermCutoff, &h.hrec_n, &h.hrec_q);
    if (tm)
        std::fprintf(stderr, "  hess sets: direct %.3f ms (%zu points), reciprocal %.3f ms (%zu)\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(), h.hdir_w.size(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(),
                     h.hrec_n.size() / h.d);
    h.has_hess = 1;
}

void build_deriv_sets(const HostCtx& h, int order, std::vector<double>* dir_n, std::vector<double>* rec_n) {
    std::vector<double> dz, dw, rq;
    enumerate_direct(h, order, 1e-20, dir_n, &dz, &dw);
    enumerate_reciprocal(h, h.k.s + order, 1e-20, rec_n, &rq);
}

// Rigorous lower bound of x = c |k + q|^2 over k in the BZ box and q != 0:
// ||kappa + n||_inf >= 1/2 gives |B (kappa + n)|^2 >= sigma_min(B)^2 / 4.
double table_x_lo(const HostCtx& h) {
    const int d = h.d;
    // smallest eigenvalue of B^T B by cyclic Jacobi
    ld m[kMaxDim][kMaxDim];
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            ld s = 0.0L;
            for (int r = 0; r < d; ++r) s += ld(h.B[r * d + i]) * h.B[r * d + j];
            m[i][j] = s;
        }
    for (int sweep = 0; sweep < 60; ++sweep) {
        ld off = 0.0L;
        for (int p = 0; p < d; ++p)
            for (int q = p + 1; q < d; ++q) off += m[p][q] * m[p][q];
        if (off < 1e-36L) break;
        for (int p = 0; p < d; ++p)
            for (int q = p + 1; q < d; ++q) {
                if (m[p][q] == 0.0L) continue;
                ld theta = (m[q][q] - m[p][p]) / (2.0L * m[p][q]);
                ld tt = (theta >= 0 ? 1.0L : -1.0L) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0L));
                ld cs = 1.0L / std::sqrt(tt * tt + 1.0L), sn = tt * cs;
                for (int r = 0; r < d; ++r) {
                    ld a1 = m[r][p], a2 = m[r][q];
                    m[r][p] = cs * a1 - sn * a2;
                    m[r][q] = sn * a1 + cs * a2;
                }
                for (int r = 0; r < d; ++r) {
                    ld a1 = m[p][r], a2 = m[q][r];
                    m[p][r] = cs * a1 - sn * a2;
                    m[q][r] = sn * a1 + cs * a2;
                }
            }
    }
    ld lmin = m[0][0];
    for (int i = 1; i < d; ++i) lmin = std::min(lmin, m[i][i]);
    return double(ld(h.k.c) * lmin / 4.0L * (1.0L - 1e-9L));
}

// ---------------------------------------------------------------------------
// Piecewise Chebyshev-interpolant tables of f_j(x) = scale_j * E_{p_j}(x).
namespace {

struct Fn {
    ld p, scale;
    ld operator()(ld x) const { return scale * expint<ld>(p, x); }
};

// Chebyshev interpolation at kNC first-kind nodes, converted to monomials in delta = tau / 2
// in [-1/2, 1/2] (c_j tau^j = (2^j c_j) delta^j: exact rescaling, same conditioning; the device
// gets delta = (fs - 1/2) - floor(fs) without the extra 2 x - 1 step).
// Chebyshev nodes, the cosine (DCT) matrix and the monomial coefficients of T_k, computed once.
template <int N> struct ChebConsts {
    ld tau[N];
    ld cosm[N][N];   // cos(pi k (i + 1/2) / N)
    ld tk[N][N];     // T_k(tau) = sum_j tk[k][j] tau^j
    ChebConsts() {
        for (int i = 0; i < N; ++i) tau[i] = std::cos(kPiL * (i + 0.5L) / N);
        for (int k = 0; k < N; ++k)
            for (int i = 0; i < N; ++i) cosm[k][i] = std::cos(kPiL * k * (i + 0.5L) / N);
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j) tk[k][j] = 0.0L;
        tk[0][0] = 1.0L;
        if (N > 1) tk[1][1] = 1.0L;
        for (int k = 2; k < N; ++k)
            for (int j = 0; j < N; ++j)
                tk[k][j] = (j > 0 ? 2.0L * tk[k - 1][j - 1] : 0.0L) - tk[k - 2][j];
    }
};
template <int N> const ChebConsts<N>& cheb() {
    static const ChebConsts<N> c;
    return c;
}

template <int N> void fit_piece(const Fn& f, ld x0, ld x1, double* out) {
    const ChebConsts<N>& C = cheb<N>();
    ld fv[N];
    ld mid = 0.5L * (x0 + x1), half = 0.5L * (x1 - x0);
    for (int i = 0; i < N; ++i) fv[i] = f(mid + half * C.tau[i]);
    ld ak[N];
    for (int k = 0; k < N; ++k) {
        ld s = 0.0L;
        for (int i = 0; i < N; ++i) s += fv[i] * C.cosm[k][i];
        ak[k] = (k == 0 ? 1.0L : 2.0L) * s / N;
    }
    for (int j = 0; j < N; ++j) {
        ld c = 0.0L;
        for (int k = 0; k < N; ++k) c += ak[k] * C.tk[k][j];
        out[j] = double(std::ldexp(c, j));
    }
}

// evaluate exactly as the device does (Estrin form, double)
ld eval_piece(const double* c, ld tau) { return estrin(c, tau_powers(double(tau) * 0.5)); }
ld eval_piece_lo(const double* c, ld tau) { return estrin_lo(c, tau_powers(double(tau) * 0.5)); }

}  // namespace

double fit_piece_fn(const std::function<long double(long double)>& f, long double x0, long double x1, double* out) {
    const ChebConsts<kNC>& C = cheb<kNC>();
    ld fv[kNC];
    const ld mid = 0.5L * (x0 + x1), half = 0.5L * (x1 - x0);
    for (int i = 0; i < kNC; ++i) fv[i] = f(mid + half * C.tau[i]);
    ld ak[kNC];
    for (int k = 0; k < kNC; ++k) {
        ld s = 0.0L;
        for (int i = 0; i < kNC; ++i) s += fv[i] * C.cosm[k][i];
        ak[k] = (k == 0 ? 1.0L : 2.0L) * s / kNC;
    }
    for (int j = 0; j < kNC; ++j) {
        ld c = 0.0L;
        for (int k = 0; k < kNC; ++k) c += ak[k] * C.tk[k][j];
        out[j] = double(std::ldexp(c, j));
    }
    // worst absolute error at 21 points, evaluated in the device's order
    double worst = 0.0;
    for (int i = 0; i <= 20; ++i) {
        const ld tau = -1.0L + 2.0L * i / 20.0L;
        worst = std::max(worst, double(std::fabs(eval_piece(out, tau) - f(mid + half * tau))));
    }
    return worst;
}

void build_table(const double* p, const double* scale, int nfunc, double c, double x_lo,
                 double rfac_pref, HostTable* out, double poly_pow, double term_cutoff) {
    // weight of a term relative to the unit scale: (1 + 4x)^poly_pow covers the |y|^2 (Hessian)
    // or |2y|^m (order-m derivative) factors multiplying the tabulated functions
    auto wfac = [poly_pow](ld x) { return std::pow(1.0L + 4.0L * x, ld(poly_pow)); };
    (void)c;
    out->nfunc = nfunc;
    for (int j = 0; j < nfunc; ++j) {
        out->p[j] = p[j];
        out->scale[j] = scale[j];
    }
    std::vector<Fn> fns;
    for (int j = 0; j < nfunc; ++j) fns.push_back(Fn{ld(p[j]), ld(scale[j])});
    // upper end: every function (times the |y|^2 factor of the Hessian terms) is
    // below `cutoff` (default 1e-18, the reference's term cutoff L/epstein.py:51) of the unit
    // scale; terms past it are exactly
    // zero in the kernel and culled per warp.
    ld cutoff = ld(term_cutoff);
    if (const char* e = std::getenv("LATSUM_TABLE_CUTOFF")) cutoff = std::strtold(e, nullptr);
    const ld hb = kBinWidth;
    ld x_hi = x_lo;
    for (int b = 0; b < 1000; ++b) {
        ld x = ld(x_lo) + hb * b;
        ld worst = 0.0L;
        for (const Fn& f : fns) worst = std::max(worst, std::fabs(f(x)) * wfac(x));
        x_hi = x;
        if (worst * std::fabs(ld(rfac_pref)) < cutoff && x > 8.0L) break;
    }
    const int nbins = int(std::lround((x_hi - ld(x_lo)) / hb));
    out->x_lo = x_lo;
    out->inv_hb = double(1.0L / hb);
    out->nbins = nbins;
    out->x_hi = double(ld(x_lo) + hb * nbins);
    out->dir.assign(nbins, 0);
    out->coef.clear();
    out->max_rel_err = 0.0;
    // Bins are independent: fit them on all host cores, then concatenate in order.  A bin gets
    // the cheap degree-kDegLo pieces when their error, weighted like the cutoff test (times
    // |rfac pref| (1 + 4x)), stays below kLoBudget x cutoff everywhere in the bin -- far-out terms
    // (most of the reciprocal ball: E_p decays like e^-x) need only absolute accuracy at the
    // level of the terms the cutoff already drops.  Otherwise degree kDeg pieces are fitted to
    // 6e-16 relative error.  Both are checked at 11 points per piece with the device's exact
    // evaluation order.
    struct BinFit {
        int level = kDirectMarker;
        int lo = 0;
        double err = 0.0;
        std::vector<double> coefs;   // [sub][func][kNCP] fit arrays
    };
    const ld lo_budget = kLoBudget * cutoff / std::max(std::fabs(ld(rfac_pref)), 1e-300L);
    std::vector<BinFit> fits(nbins);
    const int kMaxLevel = 8;
    auto try_fit = [&](ld b0, int level, bool lo, BinFit* bf) -> bool {
        const int nsub = 1 << level;
        std::vector<double> coefs(size_t(nsub) * nfunc * kNCP, 0.0);
        double worst_err = 0.0;
        for (int sidx = 0; sidx < nsub; ++sidx) {
            ld x0 = b0 + hb * sidx / nsub, x1 = b0 + hb * (sidx + 1) / nsub;
            for (int j = 0; j < nfunc; ++j) {
                double* cf = &coefs[(size_t(sidx) * nfunc + j) * kNCP];
                if (lo) fit_piece<kDegLo + 1>(fns[j], x0, x1, cf);
                else fit_piece<kNC>(fns[j], x0, x1, cf);
                for (int tidx = 0; tidx <= 10; ++tidx) {
                    ld tau = -1.0L + 2.0L * tidx / 10.0L;
                    ld xx = 0.5L * (x0 + x1) + 0.5L * (x1 - x0) * tau;
                    ld truth = fns[j](xx);
                    ld approx = lo ? eval_piece_lo(cf, tau) : eval_piece(cf, tau);
                    if (lo) {
                        if (std::fabs(approx - truth) * wfac(xx) > lo_budget) return false;
                    } else {
                        double rel = double(std::fabs(approx - truth) / std::max(std::fabs(truth), 1e-300L));
                        worst_err = std::max(worst_err, rel);
                        if (rel > 6e-16) return false;
                    }
                }
            }
        }
        bf->level = level;
        bf->lo = lo ? 1 : 0;
        bf->err = worst_err;
        bf->coefs.swap(coefs);
        return true;
    };
    // subdivision levels allowed for low-degree bins (LATSUM_LO_LEVELS): finer degree-4 pieces
    // beat degree-8 ones (fcc ATM: levels 1 -> 12.55 ms, 2 -> 12.46, 3 -> 12.39, 4 -> 12.24,
    // 5 -> 12.20 with 111 KB of tables); 4 balances kernel time against host fitting time
    int kLoMaxLevel = 4;
    if (const char* e = std::getenv("LATSUM_LO_LEVELS")) kLoMaxLevel = std::atoi(e);
    const char* lo_env = std::getenv("LATSUM_TABLE_LO");
    const bool use_lo = !(lo_env && std::atoi(lo_env) == 0);
    auto fit_bin = [&](int b) {
        const ld b0 = ld(x_lo) + hb * b;
        BinFit& bf = fits[b];
        if (use_lo)
            for (int level = 0; level <= kLoMaxLevel; ++level)
                if (try_fit(b0, level, true, &bf)) return;
        for (int level = 0; level <= kMaxLevel; ++level)
            if (try_fit(b0, level, false, &bf)) return;
        bf.level = kDirectMarker;  // evaluate E_p directly in this bin
    };
    parallel_for(nbins, 1, [&](int64_t b) { fit_bin(int(b)); });
    // Low-degree bins form a suffix [lo_start, nbins) (so the kernel can split its q loop by x
    // without per-lane layout checks); low-degree fits before it are redone at degree kDeg.
    int lo_start = nbins;
    while (lo_start > 0 && fits[lo_start - 1].level != kDirectMarker && fits[lo_start - 1].lo) --lo_start;
    {
        std::vector<int> redo;
        for (int b = 0; b < lo_start; ++b)
            if (fits[b].lo) redo.push_back(b);
        parallel_for(int64_t(redo.size()), 1, [&](int64_t i) {
            const int b = redo[size_t(i)];
            const ld b0 = ld(x_lo) + hb * b;
            BinFit& bf = fits[b];
            bf = BinFit();
            for (int level = 0; level <= kMaxLevel; ++level)
                if (try_fit(b0, level, false, &bf)) return;
            bf.level = kDirectMarker;
        });
    }
    out->lo_start = lo_start;
    // Direct (unfitted) bins must form a prefix: the kernel's conversion-free floor may step one
    // piece past a bin's last piece at an exact bin boundary, which is then the next bin's first
    // piece evaluated at the same x (delta = -1/2) -- valid only if that next bin has pieces, and
    // read in the previous bin's layout: the last high-degree bin is therefore followed by a
    // guard piece, the first low-degree piece in the high-degree layout (exact: c5..c8 = 0).
    int last_direct = -1;
    for (int b = 0; b < nbins; ++b)
        if (fits[b].level == kDirectMarker) last_direct = b;
    for (int b = 0; b < last_direct; ++b) fits[b].level = kDirectMarker;
    if (std::getenv("LATSUM_DEBUG_TABLE"))
        std::fprintf(stderr, "table: p0 %.3f nfunc %d x_lo %.4f x_hi %.3f bins %d direct-bins %d (up to x = %.3f)\n",
                     p[0], nfunc, x_lo, double(out->x_hi), nbins, last_direct + (last_direct >= 0 ? 1 : 0),
                     double(ld(x_lo) + hb * (last_direct + 1)));
    size_t off = 0;
    out->npieces = 0;
    out->n_lo_bins = 0;
    for (int b = 0; b < nbins; ++b) {
        const BinFit& bf = fits[b];
        if (b == lo_start && b > 0 && fits[b - 1].level != kDirectMarker && !fits[b - 1].lo) {
            const int ps = piece_stride(nfunc);
            const size_t base = out->coef.size();
            out->coef.resize(base + ps, 0.0);
            for (int j = 0; j < nfunc; ++j) {
                const double* cf = &bf.coefs[size_t(j) * kNCP];  // first sub-piece of bin b
                for (int m = 0; m <= kDegLo; ++m) out->coef[base + j * 8 + m] = cf[m];
            }
            off += size_t(ps);
        }
        if (bf.level == kDirectMarker) {
            out->dir[b] = kDirectMarker;
            continue;
        }
        if (bf.lo) out->n_lo_bins += 1;
        else out->max_rel_err = std::max(out->max_rel_err, bf.err);
        // entry: element offset of the bin's first piece, low-degree flag, subdivision level
        out->dir[b] = int((off << 5) | (size_t(bf.lo) << 4) | size_t(bf.level));
        // fit arrays [sub][func][kNCP] -> device layout [sub][piece_stride(nfunc)]
        const int ps = bf.lo ? piece_stride_lo(nfunc) : piece_stride(nfunc);
        const int nc = bf.lo ? kDegLo : 8;  // leading coefficients per function
        for (int sidx = 0; sidx < (1 << bf.level); ++sidx) {
            const size_t base = out->coef.size();
            out->coef.resize(base + ps, 0.0);
            for (int j = 0; j < nfunc; ++j) {
                const double* cf = &bf.coefs[(size_t(sidx) * nfunc + j) * kNCP];
                for (int m = 0; m < nc; ++m) out->coef[base + j * nc + m] = cf[m];
                if (bf.lo) out->coef[base + nfunc * nc + j] = cf[kDegLo];
                else if (kDeg == 8) out->coef[base + nfunc * 8 + j] = cf[8];
            }
            off += size_t(ps);
            out->npieces += 1;
        }
    }
    if (off >= (size_t(1) << 26)) fail(1, "coefficient table too large");
}

// Persistent worker pool (created on first use, never torn down: process exit ends the blocked
// workers).  Several callers may have jobs queued at once (plan builds on different Python
// threads, the table fit on its async thread); each caller also works on its own job, so nested
// or concurrent calls always progress.
namespace {
struct PJob {
    const std::function<void(int64_t)>* body;
    int64_t n, grain;
    std::atomic<int64_t> next{0}, done{0};
};
struct Pool {
    std::mutex m;
    std::condition_variable cv, cv_done;
    std::deque<PJob*> q;
    explicit Pool(unsigned workers) {
        for (unsigned i = 0; i < workers; ++i) std::thread([this] { run(); }).detach();
    }
    void run() {
        std::unique_lock<std::mutex> l(m);
        for (;;) {
            cv.wait(l, [this] { return !q.empty(); });
            PJob* j = q.front();
            const int64_t n = j->n, grain = j->grain;
            const int64_t b = j->next.fetch_add(grain);
            if (b >= n) {
                q.pop_front();  // exhausted (its caller waits for the chunks still running)
                continue;
            }
            l.unlock();
            const int64_t e = std::min(n, b + grain);
            for (int64_t i = b; i < e; ++i) (*j->body)(i);
            const bool last = j->done.fetch_add(e - b) + (e - b) == n;
            l.lock();
            if (last) cv_done.notify_all();
        }
    }
};
Pool& pool(unsigned workers) {
    static Pool* p = new Pool(workers);
    return *p;
}
}  // namespace

void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t)>& body) {
    grain = std::max<int64_t>(1, grain);
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n < 2 * grain || n < 8 || nth == 1) {
        for (int64_t i = 0; i < n; ++i) body(i);
        return;
    }
    Pool& P = pool(nth - 1);
    PJob job;
    job.body = &body;
    job.n = n;
    job.grain = grain;
    {
        std::lock_guard<std::mutex> l(P.m);
        P.q.push_back(&job);
    }
    P.cv.notify_all();
    for (int64_t b = job.next.fetch_add(grain); b < n; b = job.next.fetch_add(grain)) {
        const int64_t e = std::min(n, b + grain);
        for (int64_t i = b; i < e; ++i) body(i);
        job.done.fetch_add(e - b);
    }
    std::unique_lock<std::mutex> l(P.m);
    P.cv_done.wait(l, [&] { return job.done.load() == n; });
    for (auto it = P.q.begin(); it != P.q.end(); ++it)
        if (*it == &job) {
            P.q.erase(it);
            break;
        }
}

// Gauss-Legendre nodes/weights on [-1, 1] by Newton iteration on P_n (long double).
void gauss_legendre(int n, std::vector<double>* xs, std::vector<double>* ws) {
    xs->assign(n, 0.0);
    ws->assign(n, 0.0);
    // Bonnet recurrence P_k = a_k x P_{k-1} - b_k P_{k-2} with a_k = (2k-1)/k, b_k = (k-1)/k
    // precomputed (no division per step); the nodes are symmetric, so only the upper half is
    // iterated (Newton from the Tricomi guess), x_{n-1-i} = -x_i
    std::vector<ld> ak(size_t(n) + 1, 0.0L), bk(size_t(n) + 1, 0.0L);
    for (int k = 2; k <= n; ++k) {
        ak[size_t(k)] = (2.0L * k - 1.0L) / k;
        bk[size_t(k)] = (k - 1.0L) / k;
    }
    auto legendre = [&](ld x, ld* pn, ld* pn1) {
        ld p0 = 1.0L, p1 = x;
        for (int k = 2; k <= n; ++k) {
            const ld p2 = ak[size_t(k)] * x * p1 - bk[size_t(k)] * p0;
            p0 = p1;
            p1 = p2;
        }
        if (n == 1) {
            p1 = x;
            p0 = 1.0L;
        }
        *pn = p1;
        *pn1 = p0;
    };
    for (int i = 0; i < (n + 1) / 2; ++i) {
        ld x = std::cos(kPiL * (i + 0.75L) / (n + 0.5L));
        ld p1 = 0.0L, p0 = 0.0L, dp = 0.0L;
        for (int it = 0; it < 100; ++it) {
            legendre(x, &p1, &p0);
            dp = n * (x * p1 - p0) / (x * x - 1.0L);
            const ld dx = p1 / dp;
            x -= dx;
            // relative test: an absolute one never triggers near +-1 in long double
            if (std::fabs(dx) <= 4e-19L * std::fabs(x) || it > 20) break;
        }
        if (2 * i + 1 == n) x = 0.0L;  // the middle node of an odd rule
        legendre(x, &p1, &p0);
        dp = n * (x * p1 - p0) / (x * x - 1.0L);
        const double w = double(2.0L / ((1.0L - x * x) * dp * dp));
        // ascending order (numpy leggauss order)
        (*xs)[n - 1 - i] = double(x);
        (*ws)[n - 1 - i] = w;
        if (2 * i + 1 != n) {
            (*xs)[i] = -double(x);
            (*ws)[i] = w;
        }
    }
}

}  // namespace lz

namespace lz {

// ---------------------------------------------------------------------------
// Partial derivatives of Z_reg at k = 0 (reference: EpsteinContext.reg_derivatives,
// L/epstein.py:328-415).  Derived here from the Gaussian representation
//     F(|y|^2) = rho^{-s} Gamma(s, c rho) = int_c^inf tau^{s-1} exp(-tau |y|^2) d tau,
// whose y-derivatives are Hermite polynomials:
//     d^alpha F = (-1)^|alpha| sum_j prod_i h(alpha_i, j_i) y^{alpha-2j} |y|^{-2(s+p)} Gamma(s+p, c|y|^2),
//     p = |alpha| - |j|,  h(n, j) = (-1)^j n! 2^{n-2j} / (j! (n-2j)!),
// the direct sum gives (-1)^{|alpha|/2} (2 pi)^|alpha| 2 sum_z w_z z^alpha, and the
// q = 0 regular part t0_reg(rho) = sum_n a_n rho^n gives a_n n!/prod (alpha_i/2)! prod alpha_i!.
// All sums are compensated in long double.
namespace {

struct Acc {  // Neumaier summation in long double
    ld s = 0.0L, c = 0.0L;
    void add(ld x) {
        ld t = s + x;
        c += (std::fabs(s) >= std::fabs(x)) ? (s - t) + x : (x - t) + s;
        s = t;
    }
    ld value() const { return s + c; }
};

ld factl(int n) {
    ld f = 1.0L;
    for (int i = 2; i <= n; ++i) f *= i;
    return f;
}

ld hermite_coef(int n, int j) {
    return ((j & 1) ? -1.0L : 1.0L) * factl(n) * std::pow(2.0L, ld(n - 2 * j)) / (factl(j) * factl(n - 2 * j));
}

// rho-series coefficient a_n of t0_reg (L/epstein.py:328-345)
ld t0_series_coeff(const CtxConst& k, int n) {
    const ld c = kPiL / ld(k.split);
    if (k.branch == kLogCase) {
        const int m = k.log_m;
        ld val = 0.0L;
        if (n == m) val += std::log(ld(k.split)) - ld(kEulerGamma);
        if (n > m) {
            const int l = n - m;
            val += ((l + 1) % 2 ? -1.0L : 1.0L) * std::pow(c, ld(l)) / (ld(l) * factl(l));
        }
        ld acc = 0.0L;
        for (int j = std::max(0, m - n - 1); j < m; ++j) acc += factl(j) / factl(n - m + j + 1);
        val += (((n - m) % 2 != 0) ? -1.0L : 1.0L) * std::pow(c, ld(n - m)) * acc;
        return ((m % 2) ? -1.0L : 1.0L) / factl(m) * val;
    }
    const ld s = k.s;
    return -std::pow(c, s + n) * ((n % 2) ? -1.0L : 1.0L) / (factl(n) * (s + n));
}

void enumerate_alphas(int d, int total, std::vector<int>& cur, std::vector<int>* out) {
    if (int(cur.size()) == d - 1) {
        cur.push_back(total);
        out->insert(out->end(), cur.begin(), cur.end());
        cur.pop_back();
        return;
    }
    for (int h = 0; h <= total; ++h) {
        cur.push_back(h);
        enumerate_alphas(d, total - h, cur, out);
        cur.pop_back();
    }
}

}  // namespace

long double t0_coeff(const CtxConst& k, int n) { return t0_series_coeff(k, n); }

void build_reg_derivatives(const HostCtx& h, int order, std::vector<int>* alphas, std::vector<double>* vals) {
    const int d = h.d;
    alphas->clear();
    vals->clear();
    for (int total = 0; total <= order; total += 2) {
        std::vector<int> cur;
        enumerate_alphas(d, total, cur, alphas);
    }
    const size_t na = alphas->size() / d;
    vals->assign(na, 0.0);
    if (h.k.branch == kTrivial) {
        for (size_t i = 0; i < na; ++i) {
            int tot = 0;
            for (int a = 0; a < d; ++a) tot += (*alphas)[i * d + a];
            (*vals)[i] = tot == 0 ? h.k.const_value : 0.0;
        }
        return;
    }
    // widened point sets (L/epstein.py:376-377): z^alpha and shifted gamma orders
    std::vector<double> dn, dz, dw, rn, rq;
    enumerate_direct(h, order, 1e-20, &dn, &dz, &dw);
    enumerate_reciprocal(h, h.k.s + order, 1e-20, &rn, &rq);
    const CtxConst& k = h.k;
    const ld c = kPiL / ld(k.split), s = k.s;
    const size_t nd = dw.size(), nr = rq.size() / d;
    // long-double copies; reciprocal gammas per order p
    std::vector<ld> z(nd * d), q(nr * d), qn2(nr);
    for (size_t i = 0; i < nd; ++i)
        for (int a = 0; a < d; ++a) {
            ld v = 0.0L;
            for (int b = 0; b < d; ++b) v += ld(h.A[a * d + b]) * dn[i * d + b];
            z[i * d + a] = v;
        }
    std::vector<ld> wz(nd);
    for (size_t i = 0; i < nd; ++i) {
        ld r2 = 0.0L;
        for (int a = 0; a < d; ++a) r2 += z[i * d + a] * z[i * d + a];
        wz[i] = upper_gamma<ld>(ld(k.nu) / 2.0L, kPiL * ld(k.split) * r2) * std::pow(r2, -ld(k.nu) / 2.0L);
    }
    for (size_t i = 0; i < nr; ++i) {
        ld r2 = 0.0L;
        for (int a = 0; a < d; ++a) {
            ld v = 0.0L;
            for (int b = 0; b < d; ++b) v += ld(h.B[a * d + b]) * rn[i * d + b];
            q[i * d + a] = v;
            r2 += v * v;
        }
        qn2[i] = r2;
    }
    std::vector<std::vector<ld>> gam(order + 1, std::vector<ld>(nr));
    for (int p = 0; p <= order; ++p)
        for (size_t i = 0; i < nr; ++i)
            gam[p][i] = upper_gamma<ld>(s + p, c * qn2[i]) * std::pow(qn2[i], -(s + p));
    auto ipow = [](ld x, int e) {
        ld r = 1.0L;
        for (int i = 0; i < e; ++i) r *= x;
        return r;
    };
    for (size_t ia = 0; ia < na; ++ia) {
        const int* al = &(*alphas)[ia * d];
        int total = 0;
        for (int a = 0; a < d; ++a) total += al[a];
        Acc parts;
        // direct space
        {
            Acc sd;
            for (size_t i = 0; i < nd; ++i) {
                ld zp = wz[i];
                for (int a = 0; a < d; ++a) zp *= ipow(z[i * d + a], al[a]);
                sd.add(zp);
            }
            parts.add(((total / 2) % 2 ? -1.0L : 1.0L) * std::pow(2.0L * kPiL, ld(total)) * 2.0L * sd.value());
        }
        if (total == 0) parts.add(ld(k.bconst));
        // reciprocal space, Hermite expansion over j with 0 <= j_i <= alpha_i / 2
        int jv[kMaxDim] = {0, 0, 0, 0};
        for (;;) {
            int jsum = 0;
            ld coef = 1.0L;
            for (int a = 0; a < d; ++a) {
                jsum += jv[a];
                coef *= hermite_coef(al[a], jv[a]);
            }
            const int p = total - jsum;
            Acc sr;
            for (size_t i = 0; i < nr; ++i) {
                ld qp = gam[p][i];
                for (int a = 0; a < d; ++a) qp *= ipow(q[i * d + a], al[a] - 2 * jv[a]);
                sr.add(qp);
            }
            parts.add(ld(k.rfac) * coef * sr.value());
            int a = 0;
            while (a < d) {
                if (++jv[a] <= al[a] / 2) break;
                jv[a] = 0;
                ++a;
            }
            if (a == d) break;
        }
        // q = 0 regular part: only all-even multi-indices survive
        bool even = true;
        for (int a = 0; a < d; ++a) even = even && (al[a] % 2 == 0);
        if (even) {
            const int n = total / 2;
            ld mult = factl(n), fac = 1.0L;
            for (int a = 0; a < d; ++a) {
                mult /= factl(al[a] / 2);
                fac *= factl(al[a]);
            }
            parts.add(ld(k.rfac) * t0_series_coeff(k, n) * mult * fac);
        }
        (*vals)[ia] = double(ld(k.pref) * parts.value());
    }
}

}  // namespace lz
