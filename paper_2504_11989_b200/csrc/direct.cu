// Truncated direct summation of three-body lattice sums on the GPU (the SPEC's
// "oracle" module): brute force over x, y in A{-L..L}^d,
//
//   kind 0:  sum' |x|^-nu1 |y-x|^-nu2 |y|^-nu3              (zeta^(3)(nu1, nu2, nu3))
//   kind 1:  (1/6) sum' U_ATM(x, y),  U_ATM = (1 + 3 cos cos cos) / (r1 r2 r3)^3
//            = [1 - 3 (d1.d2)(d2.d3)(d3.d1) / (r1 r2 r3)^2] / (r1 r2 r3)^3
//
// with x, y, x - y != 0.  This is an independent check of the Epstein-zeta
// method (no special functions, no quadrature), converging only algebraically in L.
// Layout: one thread per x; the y points stream through shared memory in tiles of
// 256 (classic tiled N-body), each thread accumulates with Neumaier compensation;
// block partials are reduced in a fixed order by reduce_kernel.
#include <cuda_runtime.h>

#include <cstdint>

namespace lz {

constexpr int kDirTile = 256;

template <int D>
__device__ __forceinline__ void box_point(int64_t idx, int64_t L, const double* __restrict__ A, double (&x)[D],
                                          bool& is_zero) {
    const int64_t w = 2 * L + 1;
    int64_t n[D];
    int64_t rem = idx;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
        n[a] = rem % w - L;
        rem /= w;
    }
    is_zero = true;
#pragma unroll
    for (int a = 0; a < D; ++a) is_zero = is_zero && n[a] == 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < D; ++b) s = fma(A[a * D + b], double(n[b]), s);
        x[a] = s;
    }
}

template <int D, int KIND>
__global__ void __launch_bounds__(kDirTile) direct_kernel(int64_t L, int64_t npts, const double* __restrict__ Ag,
                                                          double nu1, double nu2, double nu3,
                                                          double* __restrict__ partials) {
    __shared__ double A[16];
    __shared__ double ys[kDirTile][D + 1];  // y coordinates and |y|^2
    if (threadIdx.x < D * D) A[threadIdx.x] = Ag[threadIdx.x];
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * kDirTile + threadIdx.x;
    double x[D];
    bool x_zero = true;
    const bool have_x = i < npts;
    box_point<D>(have_x ? i : 0, L, A, x, x_zero);
    double r1 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) r1 = fma(x[a], x[a], r1);
    const bool live = have_x && !x_zero;
    const double l1 = live ? -0.5 * nu1 * log(r1) : 0.0;
    double s = 0.0, comp = 0.0;
    for (int64_t base = 0; base < npts; base += kDirTile) {
        __syncthreads();
        const int64_t j = base + threadIdx.x;
        if (j < npts) {
            double y[D];
            bool yz;
            box_point<D>(j, L, A, y, yz);
            double r2 = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                ys[threadIdx.x][a] = y[a];
                r2 = fma(y[a], y[a], r2);
            }
            ys[threadIdx.x][D] = yz ? 0.0 : r2;  // |y|^2 = 0 marks the excluded origin
        } else {
            ys[threadIdx.x][D] = 0.0;
        }
        __syncthreads();
        if (!live) continue;
        const int cnt = int(npts - base < kDirTile ? npts - base : kDirTile);
        double row = 0.0;
        for (int t = 0; t < cnt; ++t) {
            const double r2 = ys[t][D];
            double zv[D], r3 = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                zv[a] = ys[t][a] - x[a];
                r3 = fma(zv[a], zv[a], r3);
            }
            double term = 0.0;
            if (r2 > 0.0 && r3 > 0.0) {
                if constexpr (KIND == 1) {
                    // triangle sides d1 = x, d2 = z = y - x, d3 = -y; the cosine product of the
                    // ATM potential is -(d1.d2)(d2.d3)(d3.d1) / (r1 r2 r3)^2 (squared norms here)
                    double xz = 0.0, zy = 0.0, yx = 0.0;
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        xz = fma(x[a], zv[a], xz);
                        zy = fma(zv[a], ys[t][a], zy);
                        yx = fma(ys[t][a], x[a], yx);
                    }
                    // d1 = x, d2 = z, d3 = -y: (d1.d2)(d2.d3)(d3.d1) = (x.z)(-z.y)(-y.x) = xz zy yx
                    const double p = r1 * r2 * r3;
                    const double inv = rsqrt(p);
                    const double inv3 = inv * inv * inv;
                    term = inv3 * fma(-3.0, (xz * zy * yx) / p, 1.0);
                } else {
                    term = exp(l1 - 0.5 * (nu2 * log(r3) + nu3 * log(r2)));
                }
            }
            row += term;
        }
        // Neumaier accumulation of the tile's row sum
        const double tsum = s + row;
        comp += (fabs(s) >= fabs(row)) ? (s - tsum) + row : (row - tsum) + s;
        s = tsum;
    }
    // deterministic block reduction (fixed tree)
    __shared__ double red[kDirTile];
    red[threadIdx.x] = s + comp;
    __syncthreads();
    for (int h = kDirTile / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

template <int D, int KIND>
static cudaError_t launch_direct_t(int64_t L, int64_t npts, const double* A, const double* nus, double* partials,
                                   int64_t nblocks, cudaStream_t st) {
    direct_kernel<D, KIND><<<dim3(unsigned(nblocks)), kDirTile, 0, st>>>(L, npts, A, nus[0], nus[1], nus[2], partials);
    return cudaGetLastError();
}

cudaError_t launch_direct(int d, int kind, int64_t L, int64_t npts, const double* A, const double* nus,
                          double* partials, int64_t nblocks, cudaStream_t st) {
#define LZ_DCASE(DD, KK) \
    if (d == DD && kind == KK) return launch_direct_t<DD, KK>(L, npts, A, nus, partials, nblocks, st);
    LZ_DCASE(1, 0) LZ_DCASE(2, 0) LZ_DCASE(3, 0) LZ_DCASE(1, 1) LZ_DCASE(2, 1) LZ_DCASE(3, 1)
#undef LZ_DCASE
    return cudaErrorInvalidValue;
}

int direct_tile() { return kDirTile; }

}  // namespace lz
