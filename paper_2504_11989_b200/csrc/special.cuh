// Special functions for the Epstein-zeta hot path, shared by host and device.
//
// Everything the reference takes from scipy (L/incgamma.py:74,85,105,142:
// gammaincc, exp1) and its own upper_gamma dispatch (L/incgamma.py:97-114) is
// expressed here through ONE function, the generalized exponential integral
//
//     E_p(x) = int_1^inf e^{-x t} t^{-p} dt ,      x > 0, real p,
//
// because every quantity on the path is an E_p:
//   Gamma(s, x)                       = x^s E_{1-s}(x)
//   rho^{-s} Gamma(s, c rho)          = c^s E_{1-s}(c rho)        (reciprocal term)
//   d/drho of the above               = -c^{s+1} E_{-s}(c rho)     (Hessian terms)
//   d2/drho2                          =  c^{s+2} E_{-s-1}(c rho)
//   E_1(x) + log x                    = -gamma_E + Ein(x)          (L/incgamma.py:117-143)
//
// Templated on the real type: the host table builder instantiates it with
// long double (64-bit mantissa) so tabulated values carry ~1e-19 relative
// error; the device instantiates it with double for the few per-node terms
// that are evaluated directly (q = 0 terms near k = 0).
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define LZ_HD __host__ __device__ __forceinline__
#define LZ_HDI __host__ __device__ inline
#else
#define LZ_HD inline
#define LZ_HDI inline
#endif

namespace lz {

constexpr double kEulerGamma = 0.577215664901532860606512090082402431;
constexpr double kPi = 3.14159265358979323846264338327950288;

template <class T> struct Eps;
template <> struct Eps<double> { static constexpr double v = 1.2e-16; };
template <> struct Eps<long double> { static constexpr long double v = 6e-20L; };

template <class T> LZ_HD T labs_(T v) { return v < T(0) ? -v : v; }

// Ein(x) = sum_{n>=1} (-1)^{n+1} x^n / (n n!)  (entire), so E_1(x) + ln x = Ein(x) - gamma_E.
template <class T> LZ_HDI T ein_series(T x) {
    T term = T(1), acc = T(0);
    for (int n = 1; n < 200; ++n) {
        term *= -x / T(n);
        T c = -term / T(n);
        acc += c;
        if (labs_(c) <= Eps<T>::v * labs_(acc)) break;
    }
    return acc;
}

// Legendre continued fraction for E_p(x), modified Lentz.  Valid for every
// real p and x > 0; converges in O(1/x) iterations, so it is the large-x branch.
template <class T> LZ_HDI T expint_cf(T p, T x, int maxit) {
    using std::exp;
    const T tiny = T(1e-290);
    T b = x + p;
    T c = T(1) / tiny;
    T d = T(1) / (labs_(b) < tiny ? tiny : b);
    T h = d;
    for (int i = 1; i <= maxit; ++i) {
        T an = -T(i) * (p - T(1) + T(i));
        b += T(2);
        d = an * d + b;
        if (labs_(d) < tiny) d = tiny;
        d = T(1) / d;
        c = b + an / c;
        if (labs_(c) < tiny) c = tiny;
        T del = c * d;
        h *= del;
        if (labs_(del - T(1)) <= Eps<T>::v) break;
    }
    return h * exp(-x);
}

// Small-x series, integer order n >= 1:
//   E_n(x) = (-x)^{n-1}/(n-1)! (psi(n) - ln x) - sum_{m != n-1} (-x)^m / ((m-n+1) m!)
template <class T> LZ_HDI T expint_series_int(int n, T x) {
    using std::log;
    const int nm1 = n - 1;
    T ans = (nm1 != 0) ? T(1) / T(nm1) : (-log(x) - T(kEulerGamma));
    T fact = T(1);
    for (int i = 1; i < 400; ++i) {
        fact *= -x / T(i);
        T del;
        if (i != nm1) {
            del = -fact / T(i - nm1);
        } else {
            T psi = -T(kEulerGamma);
            for (int j = 1; j <= nm1; ++j) psi += T(1) / T(j);
            del = fact * (-log(x) + psi);
        }
        ans += del;
        if (labs_(del) <= labs_(ans) * Eps<T>::v) break;
    }
    return ans;
}

// Small-x series, non-integer order:
//   E_p(x) = Gamma(1-p) x^{p-1} - sum_{m>=0} (-x)^m / (m! (m+1-p))
template <class T> LZ_HDI T expint_series_frac(T p, T x) {
    using std::pow;
    using std::tgamma;
    T term = T(1), sum = T(0);
    for (int m = 0; m < 400; ++m) {
        T c = term / (T(m) + T(1) - p);
        sum += c;
        if (m > 2 && labs_(c) <= Eps<T>::v * labs_(sum)) break;
        term *= -x / T(m + 1);
    }
    return tgamma(T(1) - p) * pow(x, p - T(1)) - sum;
}

// E_p(x) for x > 0 and real p.  Branch structure:
//   p integer <= 0 : E_0 = e^{-x}/x and the stable recurrence E_{p} = (e^{-x} - p E_{p+1}) / x
//   p < 0 otherwise : E_{p + N} in (0, 1) and the same recurrence
//   x > 1           : continued fraction
//   p integer >= 1  : integer series
//   p near integer  : continued fraction (the series cancels catastrophically;
//                     mirrors the reference's Lentz branch, L/incgamma.py:32-55,110-111)
//   otherwise       : non-integer series
template <class T> LZ_HDI T expint_base(T p, T x) {
    using std::exp;
    using std::floor;
    T pr = floor(p + T(0.5));
    T dist = labs_(p - pr);
    if (dist < T(1e-12) && pr <= T(0)) {
        T emx = exp(-x);
        T e = emx / x;  // E_0
        for (int q = 0; q > int(pr); --q) {
            // E_{q-1} = (e^{-x} - (q-1) E_q) / x
            e = (emx - T(q - 1) * e) / x;
        }
        return e;
    }
    if (x > T(1)) return expint_cf(p, x, 100000);
    if (dist < T(1e-12)) return expint_series_int(int(pr), x);
    if (dist < T(1e-3)) return expint_cf(p, x, 100000);
    return expint_series_frac(p, x);
}

template <class T> LZ_HDI T expint(T p, T x) {
    using std::exp;
    using std::floor;
    const T pr = floor(p + T(0.5));
    if (p < T(0) && labs_(p - pr) >= T(1e-12)) {
        // non-integer p < 0: E_{p0}, p0 = p + N in (0, 1), then the stable recurrence
        // E_{q-1} = (e^{-x} + (1 - q) E_q) / x (all terms positive for q < 1).  The continued
        // fraction alone loses up to 1e-5 relative near x = 1 at p = -11.  (No recursion: device
        // code keeps a static stack size.)
        const int n = int(floor(-p)) + 1;
        const T p0 = p + T(n);
        T e = expint_base(p0, x);
        const T emx = exp(-x);
        T q = p0;
        for (int i = 0; i < n; ++i, q -= T(1)) e = (emx + (T(1) - q) * e) / x;
        return e;
    }
    return expint_base(p, x);
}

// Upper incomplete gamma Gamma(s, x) = x^s E_{1-s}(x), x > 0 (L/incgamma.py:97-114).
template <class T> LZ_HDI T upper_gamma(T s, T x) {
    using std::pow;
    return pow(x, s) * expint(T(1) - s, x);
}

// E_1(x) + ln x, the entire part of the exponential integral (L/incgamma.py:117-143).
template <class T> LZ_HDI T exp1_plus_log(T x) {
    using std::log;
    if (x < T(4)) return ein_series(x) - T(kEulerGamma);
    return expint_cf(T(1), x, 100000) + log(x);
}

}  // namespace lz
