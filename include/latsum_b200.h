/* latsum_b200 — C ABI of the B200-native Epstein-zeta hot path.
 *
 * Drop-in boundary for the reference package `latsum` (arXiv 2504.11989,
 * /root/reference/pkg/src/latsum, abbreviated L/ below).  The reference is pure
 * Python, so its "FFI" for this path is the Python methods themselves; each
 * entry point below names the reference interface it replaces.  The Python
 * mirror (paper_2504_11989_b200/) binds these with ctypes, and INTEGRATION.md
 * shows the ctypes stub a reference maintainer would add.
 *
 * Conventions
 *   - FP64 everywhere.  Plain pointers and sizes; no torch types.
 *   - Functions suffixed with nothing take DEVICE pointers and a cudaStream_t
 *     (passed as void*; NULL = legacy default stream) and are stream-ordered.
 *     Functions suffixed `_host` take HOST pointers and synchronise.
 *   - There is no CPU compute path: without a CUDA device every compute entry
 *     point returns LZ_ECUDA.  Context creation with device < 0 builds the
 *     host-side tables only (for inspection / tests).
 *   - Return codes map onto the reference's exceptions (L/errors.py:4-17,
 *     L/epstein.py:62-63,150-151,266-267,309-313):
 */
#ifndef LATSUM_B200_H
#define LATSUM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LZ_OK = 0,
    LZ_EINVAL = 1,     /* ValueError: bad argument, |nu| > 100, non-finite k       */
    LZ_EPOLE = 2,      /* PoleError: nu = d at k in the reciprocal lattice          */
    LZ_ENONFINITE = 3, /* ValueError("k contains non-finite entries")               */
    LZ_ECUDA = 4,      /* CUDA runtime failure or no device                          */
    LZ_ENCCL = 5,      /* NCCL unavailable or the collective failed (lz_allreduce_*) */
    LZ_ESHELLS = 6,    /* RuntimeError: sum did not truncate within shell budget    */
    LZ_ELATTICE = 7,   /* LatticeError: singular generator / unsupported dimension  */
    LZ_ESINGULAR = 8   /* ValueError: singular part undefined at k = 0              */
};

/* zeta flags (lz_zeta / lz_zeta_host) */
#define LZ_NO_REDUCE 1u     /* do not reduce k into the BZ box (reg_zeta semantics) */
#define LZ_REG_ONLY 2u      /* Z_reg only: drop shat/V (L/epstein.py:261-289)        */
#define LZ_SINGULAR_ONLY 4u /* shat(nu, k) only (L/epstein.py:217-231)               */

typedef struct lz_ctx lz_ctx;   /* one (lattice, nu) context, immutable            */
typedef struct lz_plan lz_plan; /* fused multi-context plan for the integral kernels */

typedef struct {
    int d;               /* 1..4 (L/lattice.py:20)                                 */
    double a[16];        /* generator A, row-major d x d, columns = basis vectors */
    double nu;           /* exponent                                              */
    double splitting;    /* <= 0: default V^{-2/d} (L/epstein.py:107)             */
    int deriv_order;     /* 0: zeta only; 2: also build the Hessian point sets;
                            -1 / -2: plan-private contexts with only the reciprocal /
                            only the Hessian sets (the ATM plan's Z_3 / Z_5)          */
} lz_ctx_params;

typedef struct {
    int d, branch, log_m, pole;   /* branch: 0 generic, 1 log_case, 2 trivial     */
    double nu, vol, split, s_rec, pref, rfac, bconst, kmax, singular_coef, const_value;
    int64_t n_dir, n_rec, n_dir_h, n_rec_h;
    double table_x_lo, table_x_hi, table_max_rel_err;
    int64_t table_pieces, table_bins;
} lz_ctx_info;

/* -- contexts: EpsteinContext.__init__ (L/epstein.py:99-122) + epstein_context (L/epstein.py:469-472) */
int lz_ctx_create(const lz_ctx_params* p, int device, lz_ctx** out);
int lz_ctx_destroy(lz_ctx* ctx);
int lz_ctx_get_info(const lz_ctx* ctx, lz_ctx_info* out);
/* Build (host) and upload (device) the evaluation tables now instead of on first use.
 * what: bit 1 = zeta tables, bit 2 = Hessian tables, bit 4 = only the Hessian point sets (what a
 * fused ATM plan needs; lets a caller enumerate them off the critical path).  table_* info
 * fields are zero until then. */
int lz_ctx_prepare(const lz_ctx* ctx, int what);
/* which: 0 dir_pts (z = A n), 1 dir_w, 2 rec_pts, 3 hdir_pts, 4 hdir_w, 5 rec_pts_h, 6 dir_n (int coords)
 * copies min(cap, size) doubles; returns the full size through *size.                        */
int lz_ctx_get_points(const lz_ctx* ctx, int which, double* dst, int64_t cap, int64_t* size);

/* -- EpsteinContext.zeta / reg_zeta / singular (L/epstein.py:217-231,261-320).
 * k: n x d row-major, out: n.  status (device int, may be NULL) gets bit 1 on a pole.
 * lanes_per_point: 0 = auto (1 for large batches, up to 32 for small ones). */
int lz_zeta(const lz_ctx* ctx, const double* k, int64_t n, double* out, uint32_t flags,
            int lanes_per_point, int* status, void* stream);
int lz_zeta_host(const lz_ctx* ctx, const double* k, int64_t n, double* out, uint32_t flags);

/* -- Hessian d_a d_b Z_nu(k) (upper triangle, row-major: d(d+1)/2 values per point).
 * The polynomial-weighted zeta M_ab(k) = sum' z_a z_b |z|^-nu e^{-2 pi i z.k}
 * equals -Hessian/(4 pi^2).  No reference counterpart at k != 0; the k = 0
 * analogue is EpsteinContext.reg_derivatives (L/epstein.py:347-415).
 * Requires deriv_order >= 2 at context creation. */
int lz_zeta_hessian(const lz_ctx* ctx, const double* k, int64_t n, double* out, int lanes_per_point,
                    void* stream);
int lz_zeta_hessian_host(const lz_ctx* ctx, const double* k, int64_t n, double* out);

/* -- fixed Duffy grid (L/quadrature.py:136-177): 2^{d-1} d cells x n_u (Gauss-Legendre
 * in t, u = t^grading / 2) x n_v^{d-1} (Gauss-Legendre on [0, 1/2]).  Nodes are generated
 * on device; each 256-node tile writes one partial per component. */
typedef struct {
    int n_u, n_v;
    int grading;         /* q >= 1 in u = u_lo + (1/2 - u_lo) t^q                     */
    int64_t tile_lo;     /* tile range of this call (multi-GPU shard); tile_hi <= 0: all */
    int64_t tile_hi;
    double u_lo;         /* 0: whole radial range; epsilon: outer part of the split
                            radial integral (L/quadrature.py:444-446)                 */
} lz_grid;
int lz_grid_tiles(int d, const lz_grid* g, int64_t* n_nodes, int64_t* n_tiles);

/* -- product of zetas on the grid: _product_on_batch + integrate_product
 * (L/quadrature.py:393-397,455-490), distinct exponents evaluated once per node
 * and raised to their multiplicity.  partials: n_tiles doubles (only the tiles
 * of [tile_lo, tile_hi) are written).  value = 2^d * sum(partials). */
/* Contexts created with device < 0 give host-only plans (inspection / tests; integrate -> LZ_ECUDA). */
int lz_plan_create_product(const lz_ctx* const* ctxs, const int* mult, int nctx, lz_plan** out);
/* -- ATM integrand [Z_3^3, tr(M_5^3)] with M_5 = -Hess Z_5/(4 pi^2): partials n_tiles x 2.
 * E_ATM = 2^d/6 * (sum_0 - 3 sum_1); zeta^(3)(3,3,3) = 2^d sum_0.  z5 needs deriv_order 2. */
int lz_plan_create_atm(const lz_ctx* z3, const lz_ctx* z5, lz_plan** out);
int lz_plan_destroy(lz_plan* plan);
typedef struct {
    int d, kind, nctx, hess, alias, n_funcs;       /* kind: 0 product, 1 ATM                    */
    int64_t n_dir, n_runs, n_rec;                  /* union point sets after truncation         */
    int64_t table_pieces, table_bins, n_t0, smem_bytes;
    double table_x_lo, table_x_hi, table_max_rel_err, r_cut, split, t0_rho_max;
} lz_plan_info;
int lz_plan_get_info(const lz_plan* plan, lz_plan_info* out);
int lz_plan_integrate(const lz_plan* plan, const lz_grid* g, double* partials, int grid_blocks,
                      void* stream);
/* product plan at arbitrary k (device pointers, stream-ordered): out[i] = prod_j Z_j(k_i)^{m_j},
 * k reduced into the cell; k in the reciprocal lattice of a pole context sets status bit 1.
 * Replaces _product_on_batch (L/quadrature.py:393-397) for the adaptive radial quadrature. */
int lz_plan_product_at(const lz_plan* plan, const double* k, int64_t n, double* out, int* status, void* stream);
/* fixed-order compensated sum of n_tiles x ncomp partials -> out[ncomp] (device) */
int lz_reduce_partials(const double* partials, int64_t n_tiles, int ncomp, double* out, void* stream);
/* fixed chunks of tile partials, the multi-GPU exchange unit: for c in [chunk_lo, chunk_hi)
 * chunk_out[c * ncomp + j] = fixed-order compensated sum of partials[t * ncomp + j] over tiles
 * t in [c * chunk_tiles, min((c + 1) * chunk_tiles, n_tiles)); other slots are not touched.  A
 * chunk sum depends only on the grid, so ranks that own whole chunks all-reduce
 * n_chunks * ncomp doubles and lz_reduce_partials over the chunk vector
 * gives the same bits for every world size.  Replaces the per-cell fsum of
 * L/quadrature.py:487-490. */
/* the library's chunking of an n_tiles grid: chunk_tiles = ceil(n_tiles / 96) tiles per chunk,
 * n_chunks = ceil(n_tiles / chunk_tiles) <= 96 chunks (96 splits evenly over 1, 2, 3, 4, 6, 8, 12,
 * 16, 24, 32, 48 ranks).  lz_plan_integrate_host reduces through the same chunks. */
int lz_chunk_layout(int64_t n_tiles, int64_t* chunk_tiles, int64_t* n_chunks);
int lz_reduce_chunks(const double* partials, int64_t n_tiles, int ncomp, int64_t chunk_tiles, int64_t chunk_lo,
                     int64_t chunk_hi, double* chunk_out, void* stream);
/* whole integral through host memory: out[ncomp] (value sums before the 2^d factor) */
int lz_plan_integrate_host(const lz_plan* plan, const lz_grid* g, double* out);

/* -- order-m derivatives at arbitrary k (the k != 0 generalisation of
 * the reference's derivative tables L/epstein.py:347-415, same Hermite expansion and point-set
 * rules): out[i * n_alpha + j] = d^alpha_j Z(k_i) for every multi-index |alpha| = order
 * (1 <= order <= 12, any d <= 4: the reference's order and dimension limits, L/epstein.py:347-353,
 * L/lattice.py:20) in the order of lz_multi_indices (L/epstein.py:426-433, head ascending).  The polynomial-weighted zeta is M^alpha = sum'_z z^alpha |z|^-nu e^{-2 pi i k.z}
 * = d^alpha Z / (-2 pi i)^order.  k is reduced into the cell; k in the reciprocal lattice sets
 * status bit 1 (LZ_EPOLE from the host entry point).  lz_zeta_derivatives takes device pointers
 * and is stream-ordered. */
int lz_multi_indices(int d, int order, int* alphas, int64_t cap, int64_t* n);
int lz_zeta_derivatives(const lz_ctx* ctx, int order, const double* k, int64_t n, double* out, int* status,
                        void* stream);
int lz_zeta_derivatives_host(const lz_ctx* ctx, int order, const double* k, int64_t n, double* out);

/* -- Taylor table of Z_reg at k = 0: EpsteinContext.reg_derivatives (L/epstein.py:347-415).
 * Writes n multi-indices (alphas, n x d ints) with |alpha| even <= order and their values;
 * copies min(cap, n) entries, returns n through *n. */
int lz_ctx_reg_derivatives(const lz_ctx* ctx, int order, int* alphas, double* vals, int64_t cap, int64_t* n);
/* Same table computed on the context's device (deriv.cu moment kernel at k = 0, compensated sums;
 * EpsteinContext.reg_derivatives uses this one; lz_ctx_reg_derivatives is the host long-double
 * cross-check). */
int lz_ctx_reg_derivatives_device(const lz_ctx* ctx, int order, int* alphas, double* vals, int64_t cap,
                                  int64_t* n);

/* -- host special function used by the tail algebra and tests: Gamma(s, x), x > 0 */
double lz_upper_gamma(double s, double x);

/* -- truncated direct summation over x, y in A{-L..L}^d (d <= 3), the SPEC's oracle module
 * (SPEC.md:354-406): kind 0 -> sum' |x|^-nu0 |y-x|^-nu1 |y|^-nu2,
 * kind 1 -> the ATM energy (1/6) sum' U_ATM(x, y).  max_pairs > 0 guards the (2L+1)^{2d} pair
 * count (SPEC guard 1e10 on a CPU; a B200 does ~1e11 pairs/s).  Synchronous, result on host. */
int lz_direct_sum3(int device, int d, const double* a, int64_t L, int kind, const double* nus, double max_pairs,
                   double* out);

/* -- diagnostics */
int lz_fp64_peak(int device, double* tflops_out, double* ms_out);  /* DFMA-chain probe on `device` */
/* bytes the library itself copied host->device and device->host since the last reset (every
 * cudaMemcpy* it issues: context / plan tables, grid node arrays, _host entry points' inputs and
 * results).  reset != 0 zeroes the counters after reading. */
int lz_transfer_stats(int64_t* h2d_bytes, int64_t* d2h_bytes, int reset);
/* free the library's process-wide device caches (quadrature node arrays, host-entry arenas,
 * tile scratch) so that the next call starts cold; contexts and plans the caller still holds
 * are untouched.  Synchronises the device first.  device < 0: every device. */
int lz_release_caches(int device);

/* -- multi-GPU: sum the slot-disjoint tile partials of every rank in place (SURVEY.md 8(b)
 * lz_allreduce_partials; replaces the reference's per-cell thread pool reduction,
 * L/quadrature.py:475-488, and its fsum of panel results, L/quadrature.py:236).  One
 * ncclAllReduce(double, sum) of n values on `stream` over the caller's communicator
 * (`nccl_comm` is an ncclComm_t, e.g. ProcessGroupNCCL._comm_ptr()).  NCCL is resolved at run
 * time from the copy already loaded in the process (the one that created the communicator), so
 * the library has no link-time NCCL dependency.  Returns LZ_ENCCL when NCCL is unavailable or
 * the collective fails. */
int lz_allreduce_partials(double* partials, int64_t n, void* nccl_comm, void* stream);
int lz_device_count(int* n);
const char* lz_strerror(int code);
const char* lz_last_error(void);   /* thread-local message of the last failure */
const char* lz_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LATSUM_B200_H */
