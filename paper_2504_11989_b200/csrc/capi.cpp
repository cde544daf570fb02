// extern "C" boundary of latsum_b200 (see include/latsum_b200.h).
//
// Owns the host/device lifetime of contexts and fused plans: builds the host
// tables (context.cpp), uploads them once, and launches the kernels
// (kernels.cu) on the caller's stream.  No CPU compute path exists: every
// compute entry point needs a CUDA device.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <array>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <future>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/latsum_b200.h"
#include "lz_internal.h"
#include "special.cuh"

namespace lz {
bool atm_needs_wpart(const DevPlan& P, const DevGrid& g);
cudaError_t launch_product_at(const DevPlan& P, int4 mult, const double* k, int64_t n, double* out, int G,
                              int* status, cudaStream_t st);
cudaError_t launch_batch(const DevPlan& P, bool hess, const double* k, int64_t n, double* out, uint32_t flags,
                         int G, int* status, cudaStream_t st);
cudaError_t launch_product(const DevPlan& P, const DevGrid& g, const int* mult, double* partials,
                           int grid_blocks, cudaStream_t st);
cudaError_t launch_atm(const DevPlan& P, const DevGrid& g, double* partials, int grid_blocks,
                       cudaStream_t st);
cudaError_t launch_reduce(const double* partials, int64_t n_tiles, int ncomp, double* out, cudaStream_t st);
cudaError_t launch_chunks(const double* partials, int64_t n_tiles, int ncomp, int64_t chunk, int64_t c_lo,
                          int64_t c_hi, double* chunk_out, cudaStream_t st);
cudaError_t launch_deriv(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st);
cudaError_t launch_deriv_g(const DevDeriv& P, const double* k, int64_t n, double* out, int* status, cudaStream_t st);
int deriv_count(int d, int order);
int deriv_nfunc(int order);
cudaError_t launch_probe(double* scratch, int iters, int blocks, int threads, cudaStream_t st);
cudaError_t launch_direct(int d, int kind, int64_t L, int64_t npts, const double* A, const double* nus,
                          double* partials, int64_t nblocks, cudaStream_t st);
int direct_tile();

}  // namespace lz

using lz::Error;

namespace {

thread_local std::string g_last_error;

int set_err(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error{LZ_ECUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Kernel launches: the launch status, and with LATSUM_SYNC_DEBUG=1 the completion of the launch
// on its stream (a fault is then reported by the launch that caused it, not by a later sync).
void check_launch(cudaError_t e, const char* what, cudaStream_t st) {
    check_cuda(e, what);
    static const bool dbg = std::getenv("LATSUM_SYNC_DEBUG") != nullptr;
    if (dbg) {
        const cudaError_t f = cudaStreamSynchronize(st);
        if (f != cudaSuccess) throw Error{LZ_ECUDA, std::string("after ") + what + ": " + cudaGetErrorString(f)};
    }
}

struct DeviceGuard {
    int old = -1;
    explicit DeviceGuard(int dev) {
        if (dev < 0) return;
        check_cuda(cudaGetDevice(&old), "cudaGetDevice");
        if (old != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
        else old = -1;
    }
    ~DeviceGuard() {
        if (old >= 0) cudaSetDevice(old);
    }
};

// bytes this library copied across PCIe (lz_transfer_stats): every host<->device copy below
// goes through copy_h2d / copy_d2h
std::atomic<int64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st, bool async = true) {
    g_h2d_bytes += int64_t(bytes);
    if (async) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "h2d");
    else {
        // a pageable cudaMemcpy returns once the source is staged, not when the DMA lands; the
        // kernels run on non-blocking streams that do not order after the legacy stream, so wait
        check_cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "h2d");
        check_cuda(cudaStreamSynchronize(cudaStreamLegacy), "h2d sync");
    }
}

void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    g_d2h_bytes += int64_t(bytes);
    check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "d2h");
}

template <class T> T* upload(const std::vector<T>& v, std::vector<void*>* allocs) {
    if (v.empty()) return nullptr;
    void* p = nullptr;
    check_cuda(cudaMalloc(&p, v.size() * sizeof(T)), "cudaMalloc");
    allocs->push_back(p);
    copy_h2d(p, v.data(), v.size() * sizeof(T), nullptr, false);
    return static_cast<T*>(p);
}

void free_all(std::vector<void*>* allocs) {
    for (void* p : *allocs) cudaFree(p);
    allocs->clear();
}

// Host-side description of a fused plan before upload.
struct HostPlan {
    int d = 0, nctx = 0, hess = 0, nw = 0, alias_fp = 0;
    int dir_plain = 0;  // plain-context channels in the direct weight rows (0 for trace-Z ATM plans)
    double c = 0.0, r_cut = 0.0, r_in = 0.0, alias_ratio = 0.0;
    std::vector<double> dir_n, rec_q, rec_norm, t0c;
    std::vector<double> rq_pad;   // rec_q at the padded stride (d + 1) & ~1 (device image layout)
    // direct space: [slab records][row records][weight rows] (see build_host_plan)
    std::vector<double> direct;
    int n_slabs = 0, n_rows = 0, rows_off = 0, w_off = 0, n_wrows = 0;
    double e2[4] = {0, 0, 0, 0}, e3[4] = {0, 0, 0, 0};
    int n_t0 = 0;
    double t0_rho_max = -1.0;
    // line kernel: the Hessian's q = 0 rows (t0_reg', t0_reg'') as degree-kDeg pieces on bins of
    // kBinWidth in x = c rho over [0, c t0_rho_max] (piece_stride(2) doubles per bin)
    std::vector<double> q0tab;
    int q0_nb = 0;
    double q0_inv_h = 0.0;
    std::vector<int> run_info;   // maximal runs of consecutive n_d (plan info only)
    // line-factorised direct block (trace-Z ATM plans, d = 3; see build_line_block)
    std::vector<unsigned char> line;
    int line_K[3] = {0, 0, 0}, line_P[3] = {0, 0, 0}, line_slot_off[3] = {0, 0, 0}, line_meta_off[3] = {0, 0, 0};
    double line_sign = 1.0;
    // row-factorised direct block (trace-Z ATM plans, d = 3; see build_row_block)
    std::vector<double> row_pts;
    std::vector<int> row_idx;
    int row_on = 0, row_nJ = 0, row_PS = 0, row_NI = 0;
    int row_jmin[3] = {0, 0, 0};
    lz::HostTable tab;
    lz::CtxConst ctx[lz::kMaxCtx];
    lz::CtxConst hctx;
    double A[16], B[16];
};

using ld = long double;

// LATSUM_TIMING=1: host phase times on stderr (tuning aid for the cold end-to-end path)
struct PhaseTimer {
    const char* what;
    std::chrono::steady_clock::time_point t0;
    bool on;
    explicit PhaseTimer(const char* w) : what(w), t0(std::chrono::steady_clock::now()), on(enabled()) {}
    static bool enabled() {
        static const bool e = std::getenv("LATSUM_TIMING") != nullptr;
        return e;
    }
    ~PhaseTimer() {
        if (on)
            std::fprintf(stderr, "  %-22s %.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

// Union of integer point sets (keeps the order of the first, appends the rest).
// lattice coordinates packed into one 64-bit key (16 bits per axis, d <= 4)
uint64_t pack_key(int d, const double* n) {
    uint64_t key = 0;
    for (int a = 0; a < d; ++a) {
        const long v = std::lround(n[a]);
        if (v < -32767 || v > 32767) throw Error{LZ_EINVAL, "lattice point index out of range"};
        key = (key << 16) | uint64_t(v + 32768);
    }
    return key;
}

void union_points(int d, const std::vector<const std::vector<double>*>& sets, std::vector<double>* out) {
    out->clear();
    if (sets.size() == 1) {  // one enumerated set: its points are distinct already
        *out = *sets[0];
        return;
    }
    size_t total = 0;
    for (const auto* s : sets) total += s->size() / d;
    std::unordered_set<uint64_t> seen;
    seen.reserve(2 * total);
    out->reserve(total * d);
    for (const auto* s : sets) {
        const size_t cnt = s->size() / d;
        for (size_t i = 0; i < cnt; ++i)
            if (seen.insert(pack_key(d, &(*s)[i * d])).second)
                out->insert(out->end(), s->begin() + i * d, s->begin() + (i + 1) * d);
    }
}

// Weights of the kept direct points, one row of `nw` channels per point, found by packed key.
// `keys[i]` is the packed key of row i; the key -> row map is built on first use (the row-
// factorised ATM block reads its rows through `row_of`, the sorted order's row indices, and
// never needs it).
struct WeightMap {
    mutable std::unordered_map<uint64_t, uint32_t> idx;
    std::vector<uint64_t> keys;
    std::vector<long double> rows;
    std::vector<uint32_t> row_of;   // row of hp->dir_n[i] after the lexicographic sort
    size_t nw = 0;
    const long double* at(uint64_t key) const {
        if (idx.empty() && !keys.empty()) {
            idx.reserve(2 * keys.size());
            for (size_t i = 0; i < keys.size(); ++i) idx.emplace(keys[i], uint32_t(i));
        }
        return &rows[size_t(idx.at(key)) * nw];
    }
};

// Direct-space weight w_z = Gamma(nu/2, pi t |z|^2) |z|^-nu (L/epstein.py:139), long double.
ld direct_weight(const lz::HostCtx& h, const double* n, ld* z) {
    const int d = h.d;
    ld r2 = 0.0L;
    for (int a = 0; a < d; ++a) {
        z[a] = 0.0L;
        for (int b = 0; b < d; ++b) z[a] += ld(h.A[a * d + b]) * n[b];
        r2 += z[a] * z[a];
    }
    const ld nu = h.k.nu;
    const ld x = ld(lz::kPi) * ld(h.k.split) * r2;
    return lz::upper_gamma<ld>(nu / 2.0L, x) * std::pow(r2, -nu / 2.0L);
}

bool rec_n_empty(const std::vector<const std::vector<double>*>& sets) {
    for (const auto* v : sets)
        if (!v->empty()) return false;
    return true;
}

// Build a fused plan from plain contexts (+ optionally one Hessian context).
// Line-factorised direct block for the ATM kernel (d = 3).  The 32 lanes of a warp hold nodes
// on one line of the Duffy grid: kappa = kappa_0 + x e_a with a = the cell's pyramid axis and x
// varying per lane (kernels.cu line_direct).  Grouping the half lattice by planes n_a = m,
//   sum_n W_n cos 2 pi kappa.n = sum_m Re[e^{2 pi i x m} C_m],  C_m = sum_{n_a = m} W_n e^{2 pi i kappa_0.n},
// the C_m are warp-uniform: the warp computes them cooperatively (each lane a contiguous slice of
// one plane), reduces them through shared memory and every lane finishes with one rotation per
// plane.  Per axis the half lattice is {n : (n_a, n_b, n_c) >lex 0} (b = a+1, c = a+2 mod 3);
// planes m = 0..M get lane groups sized so that the slots per lane K = max_m ceil(s_m / L_m) is
// small.  W_n = s v v^T with v = sqrt|hscale w| z (s = the common sign), one shared array of v
// (24-byte records, the last one zero); per axis each slot holds a point index (uint16) and a
// step code: the phase moves from the lane's previous point by (0, +1) (code 0) or (+1, 1 - code)
// in (n_b, n_c).
// Returns false (no line block) when the set does not fit the kernel's fixed limits.
static bool build_line_block(HostPlan* hp, const WeightMap& wmap,
                             const double* A, long double hscale, int hidx) {
    const int d = 3;
    const bool dbg = std::getenv("LATSUM_DEBUG_LINE") != nullptr;
    auto fail = [&](const char* why) {
        if (dbg) std::fprintf(stderr, "line block: %s\n", why);
        return false;
    };
    const size_t np = hp->dir_n.size() / d;
    if (np == 0) return fail("empty direct set");
    if (np >= 65535) return fail("too many points");
    const auto t_line0 = std::chrono::steady_clock::now();
    std::vector<std::array<double, 3>> v(np);
    int sign = 0;
    for (size_t i = 0; i < np; ++i) {
        const double* n = &hp->dir_n[i * d];
        long double z[3];
        for (int a = 0; a < 3; ++a) {
            z[a] = 0.0L;
            for (int b = 0; b < 3; ++b) z[a] += (long double)A[a * 3 + b] * n[b];
        }
        const long double w = wmap.at(pack_key(d, n))[hidx] * hscale;
        const int sg = w < 0 ? -1 : 1;
        if (sign != 0 && sg != sign) return fail("mixed weight signs");
        sign = sg;
        const long double r = std::sqrt(std::fabs(w));
        for (int a = 0; a < 3; ++a) v[i][a] = double(r * z[a]);
    }
    hp->line_sign = double(sign);
    std::vector<unsigned char> out;
    auto put = [&](const void* p, size_t bytes) {
        const size_t off = (out.size() + 15) & ~size_t(15);
        out.resize(off + bytes, 0);
        std::memcpy(out.data() + off, p, bytes);
        return int(off);
    };
    const auto t_line1 = std::chrono::steady_clock::now();
    struct AxisBlock {
        std::vector<uint16_t> idx;
        std::vector<uint8_t> code, glo;
        std::vector<int32_t> init;
        int K = 0, P = 0;
    };
    AxisBlock blk[3];
    const char* why[3] = {nullptr, nullptr, nullptr};
    auto axis_job = [&](int ax) {
        const int b = (ax + 1) % 3, c = (ax + 2) % 3;
        std::vector<std::vector<std::array<long, 3>>> planes;  // (nb, nc, index) per plane m
        for (size_t i = 0; i < np; ++i) {
            long n[3];
            for (int a = 0; a < 3; ++a) n[a] = std::lround(hp->dir_n[i * d + a]);
            const bool pos = n[ax] > 0 || (n[ax] == 0 && (n[b] > 0 || (n[b] == 0 && n[c] > 0)));
            if (!pos)
                for (int a = 0; a < 3; ++a) n[a] = -n[a];
            if (size_t(n[ax]) >= planes.size()) planes.resize(size_t(n[ax]) + 1);
            planes[size_t(n[ax])].push_back({n[b], n[c], long(i)});
        }
        const int P = int(planes.size());
        if (P > lz::kLinePlanes) { why[ax] = "too many planes"; return; }
        std::vector<int> L(P, 0);
        int used = 0;
        for (int p = 0; p < P; ++p)
            if (!planes[p].empty()) L[p] = 1, ++used;
        if (used > 32) { why[ax] = "more planes than lanes"; return; }
        auto load = [&](int p) { return L[p] ? (long(planes[p].size()) + L[p] - 1) / L[p] : 0L; };
        for (; used < 32; ++used) {
            int best = 0;
            for (int p = 1; p < P; ++p)
                if (load(p) > load(best)) best = p;
            ++L[best];
        }
        long K = 0;
        for (int p = 0; p < P; ++p) K = std::max(K, load(p));
        if (dbg) {
            std::fprintf(stderr, "line block axis %d: %zu points, K %ld, planes:", ax, np, K);
            for (int p = 0; p < P; ++p) std::fprintf(stderr, " %zu/%d", planes[p].size(), L[p]);
            std::fprintf(stderr, "\n");
        }
        std::vector<uint16_t> idx(size_t(K) * 32, uint16_t(np));
        std::vector<uint8_t> code(size_t(K) * 32, 0);
        std::vector<int32_t> init(32, 0);
        std::vector<uint8_t> glo(size_t(P) + 1, 0);
        int lane = 0;
        for (int p = 0; p < P; ++p) {
            glo[p] = uint8_t(lane);
            auto& pts = planes[p];
            std::sort(pts.begin(), pts.end());
            // plane p over lanes [lane, lane + L[p]): balanced contiguous chunks of the row-major
            // (n_b, n_c) order, so consecutive slots of a lane are row neighbours or a row change
            const long sz = long(pts.size());
            for (int j = 0; j < L[p]; ++j) {
                const long lo = sz * j / L[p], hi = sz * (j + 1) / L[p];
                const int ln = lane + j;
                for (long q = lo; q < hi; ++q) {
                    const size_t sl = size_t(q - lo) * 32 + ln;
                    const auto& pt = pts[q];
                    idx[sl] = uint16_t(pt[2]);
                    if (q == lo) {
                        if (std::labs(pt[0]) > 32767 || std::labs(pt[1]) > 32767) { why[ax] = "coordinates"; return; }
                        init[ln] = int32_t((uint32_t(uint16_t(int16_t(pt[0]))) << 16) | uint16_t(int16_t(pt[1])));
                    } else {
                        const long dnb = pt[0] - pts[q - 1][0], dnc = pt[1] - pts[q - 1][1];
                        if (dnb == 0 && dnc == 1) {
                            code[sl] = 0;
                        } else if (dnb == 1 && dnc <= 0 && dnc >= -30) {
                            code[sl] = uint8_t(1 - dnc);
                        } else {
                            { why[ax] = "row step out of range"; return; }
                        }
                    }
                }
            }
            lane += L[p];
        }
        glo[P] = uint8_t(lane);
        blk[ax].idx.swap(idx);
        blk[ax].code.swap(code);
        blk[ax].glo.swap(glo);
        blk[ax].init.swap(init);
        blk[ax].K = int(K);
        blk[ax].P = P;
        };
    for (int ax = 0; ax < 3; ++ax) {
        axis_job(ax);
        if (why[ax]) return fail(why[ax]);
    }
    const auto t_line2 = std::chrono::steady_clock::now();
    // Bank-aware order of the v records: a 24-byte record at position pos starts in bank pair
    // 6 pos mod 32, i.e. its bank depends on pos mod 16.  The 32 lanes of every (axis, slot)
    // gather 32 records; residues pos mod 16 are chosen so that no residue occurs more than
    // twice in any such group where possible (two wavefronts per 8-byte gather instead of ~5.6
    // for an arbitrary order), then record i goes to pos = 16 k + residue(i).
    std::vector<int> res(np, -1), perm(np, 0);
    {
        std::vector<std::array<int, 3>> groups(np, {-1, -1, -1});  // group id per axis
        int ng = 0;
        for (int ax = 0; ax < 3; ++ax) {
            for (int q = 0; q < blk[ax].K; ++q, ++ng)
                for (int l = 0; l < 32; ++l) {
                    const int i = blk[ax].idx[size_t(q) * 32 + l];
                    if (i < int(np)) groups[size_t(i)][ax] = ng;
                }
        }
        const int cap = int((np + 15) / 16);
        std::vector<std::array<int, 16>> cnt(static_cast<size_t>(ng));
        for (auto& c16 : cnt) c16.fill(0);
        std::array<int, 16> load;
        load.fill(0);
        auto cost = [&](size_t i, int r) {
            int c = 0;
            for (int ax = 0; ax < 3; ++ax) {
                const int g = groups[i][ax];
                if (g >= 0) c += std::max(0, cnt[size_t(g)][r] + 1 - 2);
            }
            return c;
        };
        auto place = [&](size_t i, int r, int sgn) {
            for (int ax = 0; ax < 3; ++ax)
                if (groups[i][ax] >= 0) cnt[size_t(groups[i][ax])][r] += sgn;
            load[r] += sgn;
        };
        for (size_t i = 0; i < np; ++i) {
            int best = -1, bc = 0;
            for (int r = 0; r < 16; ++r) {
                if (load[r] >= cap) continue;
                const int c = cost(i, r);
                if (best < 0 || c < bc || (c == bc && load[r] < load[best])) best = r, bc = c;
            }
            res[i] = best;
            place(i, best, +1);
        }
        // one repair pass over the points that still sit in an over-full group
        for (size_t i = 0; i < np; ++i) {
            if (cost(i, res[i]) <= 0 && [&] {
                    for (int ax = 0; ax < 3; ++ax)
                        if (groups[i][ax] >= 0 && cnt[size_t(groups[i][ax])][res[i]] > 2) return false;
                    return true;
                }())
                continue;
            place(i, res[i], -1);
            int best = res[i], bc = cost(i, res[i]);
            for (int r = 0; r < 16 && bc > 0; ++r) {
                if (r == res[i] || load[r] >= cap) continue;
                const int c = cost(i, r);
                if (c < bc) best = r, bc = c;
            }
            res[i] = best;
            place(i, best, +1);
        }
        std::array<int, 16> next;
        next.fill(0);
        for (size_t i = 0; i < np; ++i) perm[i] = 16 * next[res[i]]++ + res[i];
        const int nrec = 16 * cap + 1;  // the last record (a multiple of 16) is the zero padding
        if (size_t(nrec) * 24 >= 65536) return fail("too many points");
        std::vector<double> vv(size_t(nrec) * 3, 0.0);
        for (size_t i = 0; i < np; ++i)
            for (int a = 0; a < 3; ++a) vv[size_t(perm[i]) * 3 + a] = v[i][a];
        put(vv.data(), vv.size() * sizeof(double));  // at 0
        for (int ax = 0; ax < 3; ++ax)
            for (auto& ix : blk[ax].idx) ix = uint16_t(ix < np ? perm[ix] : nrec - 1);
    }
    for (int ax = 0; ax < 3; ++ax) {
        hp->line_K[ax] = blk[ax].K;
        hp->line_P[ax] = blk[ax].P;
        // slot words: byte offset of the v record (bits 0-15) | byte offset of the step entry
        // (16 code, bits 16-24)
        std::vector<uint32_t> word(blk[ax].idx.size());
        for (size_t i = 0; i < word.size(); ++i)
            word[i] = uint32_t(blk[ax].idx[i]) * 24u | (uint32_t(blk[ax].code[i]) * 16u) << 16;
        hp->line_slot_off[ax] = put(word.data(), word.size() * sizeof(uint32_t));
        hp->line_meta_off[ax] = put(blk[ax].init.data(), blk[ax].init.size() * sizeof(int32_t));
        put(blk[ax].glo.data(), blk[ax].glo.size());          // at meta_off + 128
    }
    out.resize((out.size() + 15) & ~size_t(15), 0);
    hp->line.swap(out);
    if (PhaseTimer::enabled()) {
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "  line: records %.3f ms, lane slots %.3f ms, bank order + image %.3f ms\n",
                     ms(t_line0, t_line1), ms(t_line1, t_line2), ms(t_line2, t3));
    }
    if (dbg)
        std::fprintf(stderr, "line block: %zu points, K = %d/%d/%d, planes = %d/%d/%d, %zu bytes\n", np,
                     hp->line_K[0], hp->line_K[1], hp->line_K[2], hp->line_P[0], hp->line_P[1], hp->line_P[2],
                     hp->line.size());
    return true;
}

// Row-factorised direct block for the ATM kernel (d = 3; kernels.cu row_table_kernel / row_planes).
// With the line's kappa_0 = (0, kappa_b, kappa_c) (kappa_c = u, the radial node; kappa_b = 2 s1 u v2)
// the plane sums of build_line_block factor once more over the rows n_b = j of each plane:
//   C_m = sum_j e^{2 pi i kappa_b j} D_{m,j}(u),   D_{m,j}(u) = sum_{n_c} W_n e^{2 pi i u n_c},
// and D depends only on (axis, radial node): a small table kernel forms it once per launch for the
// grid's n_u radial nodes, and a line costs one complex multiply-add per (row, plane, channel)
// instead of one term per lattice point.  Nothing of this block is staged in shared memory, so the
// direct set may grow (smaller split, fewer reciprocal terms per node).
// Per axis the half lattice is {n : (n_a, n_b, n_c) >lex 0}; rows are stored sorted by (j, m, n_c).
// Returns false when the set does not fit the kernel's fixed limits.
static bool build_row_block(HostPlan* hp, const WeightMap& wmap, const double* A, long double hscale, int hidx) {
    const int d = 3;
    const size_t np = hp->dir_n.size() / d;
    hp->row_on = 0;
    hp->row_pts.clear();
    hp->row_idx.clear();
    if (np == 0) return false;
    std::vector<std::array<double, 3>> v(np);
    std::vector<signed char> sg(np);
    lz::parallel_for(int64_t(np), 1024, [&](int64_t i) {
        const double* n = &hp->dir_n[size_t(i) * d];
        long double z[3];
        for (int a = 0; a < 3; ++a) {
            z[a] = 0.0L;
            for (int b = 0; b < 3; ++b) z[a] += (long double)A[a * 3 + b] * n[b];
        }
        const long double w = wmap.rows[size_t(wmap.row_of[size_t(i)]) * wmap.nw + size_t(hidx)] * hscale;
        sg[size_t(i)] = w < 0 ? -1 : 1;
        const long double r = std::sqrt(std::fabs(w));
        for (int a = 0; a < 3; ++a) v[size_t(i)][a] = double(r * z[a]);
    });
    const int sign = sg[0];
    for (size_t i = 1; i < np; ++i)
        if (sg[i] != sign) return false;  // mixed weight signs
    // canonical (m = n_a, j = n_b, l = n_c) of every point per axis, then a counting sort by row
    // (j, m): the order inside a row is the points' own (only the rounding of the row sums
    // depends on it)
    std::vector<int32_t> can[3];
    long jlo[3], jhi[3];
    int planes[3];
    bool too_many[3] = {false, false, false};
    lz::parallel_for(3, 1, [&](int64_t axl) {
        const int ax = int(axl);
        const int b = (ax + 1) % 3, c = (ax + 2) % 3;
        can[ax].resize(np * 3);
        jlo[ax] = 0, jhi[ax] = 0;
        long mmax = 0;
        for (size_t i = 0; i < np; ++i) {
            long n[3];
            for (int a = 0; a < 3; ++a) n[a] = std::lround(hp->dir_n[i * d + a]);
            const bool pos = n[ax] > 0 || (n[ax] == 0 && (n[b] > 0 || (n[b] == 0 && n[c] > 0)));
            if (!pos)
                for (int a = 0; a < 3; ++a) n[a] = -n[a];
            can[ax][3 * i] = int32_t(n[ax]);
            can[ax][3 * i + 1] = int32_t(n[b]);
            can[ax][3 * i + 2] = int32_t(n[c]);
            jlo[ax] = std::min(jlo[ax], n[b]);
            jhi[ax] = std::max(jhi[ax], n[b]);
            mmax = std::max(mmax, n[ax]);
        }
        too_many[ax] = mmax + 1 > lz::kLinePlanes;
        planes[ax] = int(mmax + 1);
    });
    if (too_many[0] || too_many[1] || too_many[2]) return false;
    const int pmax = std::max(planes[0], std::max(planes[1], planes[2]));
    const int rounds = (6 * pmax + 31) / 32;
    if (rounds > lz::kRowRounds) return false;
    const int NI = 32 * rounds, PS = (NI + 5) / 6;
    long nJ = 0;
    for (int ax = 0; ax < 3; ++ax) nJ = std::max(nJ, jhi[ax] - jlo[ax] + 1);
    if (nJ > 128) return false;
    hp->row_idx.assign(size_t(3) * size_t(nJ) * size_t(PS) * 2, 0);
    hp->row_pts.assign(np * 12, 0.0);
    std::vector<int> fill(size_t(nJ) * size_t(PS));
    for (int ax = 0; ax < 3; ++ax) {
        int* idx = &hp->row_idx[size_t(ax) * size_t(nJ) * size_t(PS) * 2];
        auto slot_of = [&](size_t i) {
            return size_t(can[ax][3 * i + 1] - jlo[ax]) * size_t(PS) + size_t(can[ax][3 * i]);
        };
        for (size_t i = 0; i < np; ++i) ++idx[2 * slot_of(i) + 1];
        int start = int(size_t(ax) * np);
        for (size_t sl = 0; sl < fill.size(); ++sl) {
            idx[2 * sl] = start;
            fill[sl] = start;
            start += idx[2 * sl + 1];
        }
        for (size_t i = 0; i < np; ++i) {
            double* o = &hp->row_pts[size_t(fill[slot_of(i)]++) * 4];
            o[0] = double(can[ax][3 * i + 2]);
            for (int a = 0; a < 3; ++a) o[1 + a] = v[i][a];
        }
        hp->row_jmin[ax] = int(jlo[ax]);
        hp->line_P[ax] = planes[ax];
        hp->line_K[ax] = 0;
    }
    hp->line_sign = double(sign);
    hp->row_nJ = int(nJ);
    hp->row_PS = PS;
    hp->row_NI = NI;
    hp->row_on = 1;
    if (std::getenv("LATSUM_DEBUG_LINE"))
        std::fprintf(stderr, "row block: %zu points, planes %d/%d/%d, rows j %ld, items %d (%d rounds)\n", np,
                     planes[0], planes[1], planes[2], nJ, NI, rounds);
    return true;
}

// trace_z (ATM plans): Z_nu = tr M_{nu+2} exactly (Sum_a z_a^2 |z|^{-nu-2} = |z|^{-nu}), so the
// kernel takes Z_3 from the trace of the Hessian of Z_5 and the direct weight rows carry only the
// three Hessian moment channels (nw = 3, loaded in pairs of points); the plain context still
// supplies the shared table function (F of Z_3 = F' of Z_5 / alias_ratio) and its constants.
void build_host_plan(const std::vector<const lz::HostCtx*>& plain, const lz::HostCtx* hess, HostPlan* hp,
                     bool trace_z = false) {
    const lz::HostCtx* first = plain.empty() ? hess : plain[0];
    const int d = first->d;
    hp->d = d;
    hp->nctx = int(plain.size());
    hp->hess = hess ? 1 : 0;
    std::memcpy(hp->A, first->A, sizeof(hp->A));
    std::memcpy(hp->B, first->B, sizeof(hp->B));
    std::vector<const std::vector<double>*> dsets, rsets;
    for (const auto* c : plain) {
        if (c->k.split != first->k.split) throw Error{LZ_EINVAL, "fused contexts must share the split"};
        if (std::memcmp(c->A, first->A, sizeof(c->A)) != 0)
            throw Error{LZ_EINVAL, "fused contexts must share the lattice"};
        if (!trace_z) dsets.push_back(&c->dir_n);  // trace-Z: the direct rows carry the Hessian only
        rsets.push_back(&c->rec_n);
    }
    if (hess) {
        if (hess->k.split != first->k.split) throw Error{LZ_EINVAL, "fused contexts must share the split"};
        dsets.push_back(&hess->hdir_n);
        rsets.push_back(&hess->hrec_n);
    }
    // order: largest set first so single-context plans keep the reference order
    auto by_size = [](const std::vector<double>* a, const std::vector<double>* b) { return a->size() > b->size(); };
    std::stable_sort(dsets.begin(), dsets.end(), by_size);
    std::stable_sort(rsets.begin(), rsets.end(), by_size);
    // table functions: plain F_j = c^s E_{1-s}; Hessian F' = -c^{s+1} E_{-s}, F'' = c^{s+2} E_{-s-1}
    double p[4], sc[4];
    int nf = 0;
    double rp = 0.0;
    const ld c = ld(lz::kPi) / ld(first->k.split);
    hp->c = first->k.c;
    for (int j = 0; j < hp->nctx; ++j) {
        const lz::CtxConst& k = plain[j]->k;
        hp->ctx[j] = k;
        p[nf] = 1.0 - k.s;
        sc[nf] = double(std::pow(c, ld(k.s)));
        ++nf;
        rp = std::max(rp, std::fabs(k.rfac * k.pref));
    }
    std::memset(&hp->hctx, 0, sizeof(hp->hctx));
    hp->alias_fp = 0;
    hp->alias_ratio = 0.0;
    if (hess) {
        const lz::CtxConst& k = hess->k;
        hp->hctx = k;
        // F' = -c^{s+1} E_{-s}: when plain context 0 has s0 = s + 1 its table is the same E_p
        // (ATM: Z_3 and the Hessian of Z_5); then F' = ratio * F_0 and is not tabulated
        if (hp->nctx == 1 && std::fabs(plain[0]->k.s - (k.s + 1.0)) < 1e-14) {
            hp->alias_fp = 1;
            hp->alias_ratio = double(-std::pow(c, ld(k.s) + 1.0L) / std::pow(c, ld(plain[0]->k.s)));
        } else {
            p[nf] = -k.s;
            sc[nf] = -double(std::pow(c, ld(k.s) + 1.0L));
            ++nf;
        }
        p[nf] = -k.s - 1.0;
        sc[nf] = double(std::pow(c, ld(k.s) + 2.0L));
        ++nf;
        rp = std::max(rp, std::fabs(k.rfac * k.pref));
    }
    if (nf > 4) throw Error{LZ_EINVAL, "too many functions in one plan"};
    // the piecewise tables depend only on the contexts' constants: fit them on a helper thread
    // (which fans out over the host cores) while the point sets are prepared
    std::future<void> table_job;
    const double x_lo_tab = lz::table_x_lo(*first);
    if (!rec_n_empty(rsets))
        table_job = std::async(std::launch::async, [&hp, p, sc, nf, c, x_lo_tab, rp, trace_z] {
            lz::build_table(p, sc, nf, double(c), x_lo_tab, rp, &hp->tab, 1.0,
                            trace_z ? lz::kAtmTermCutoff : 1e-18);
        });
    // q = 0 power series (t0_reg and, for the Hessian, its rho-derivatives) and the line kernel's
    // pieces of the Hessian rows: they depend only on the contexts' constants, so they are
    // prepared on a helper thread while the point sets are merged
    std::future<void> q0_job = std::async(std::launch::async, [&]     {
        const int rows = hp->nctx + (hess ? 2 : 0);
        hp->t0c.assign(size_t(std::max(rows, 1)) * lz::kT0, 0.0);
        std::vector<ld> a(lz::kT0 + 2);
        // series region: x = c rho <= max(2, x_lo) (and never beyond the BZ box); outside it
        // the kernel uses the tables, so the alternating series never cancels by more than e^2
        const ld c_l = ld(lz::kPi) / ld(first->k.split);
        const ld x_ser = std::max(2.0L, ld(lz::table_x_lo(*first)) * 1.0001L);
        ld rho_max = std::min(ld(first->kmax) * ld(first->kmax) * (1.0L + 1e-9L), x_ser / c_l);
        int need = 0;
        bool ok = true;
        auto fill = [&](const lz::CtxConst& k, int row, int deriv) {
            for (int n = 0; n < lz::kT0 + 2; ++n) a[n] = lz::t0_coeff(k, n);
            ld big = 0.0L;
            std::vector<ld> cf(lz::kT0);
            for (int n = 0; n < lz::kT0; ++n) {
                ld v = a[n + deriv];
                for (int j = 1; j <= deriv; ++j) v *= ld(n + j);
                cf[n] = v;
                big = std::max(big, std::fabs(v) * std::pow(rho_max, ld(n)));
            }
            int used = lz::kT0;
            while (used > 1 && std::fabs(cf[used - 1]) * std::pow(rho_max, ld(used - 1)) <= 1e-19L * std::max(big, 1.0L))
                --used;
            if (used >= lz::kT0 - 2) ok = false;  // not converged within kT0 terms: disable
            need = std::max(need, used + 2);
            for (int n = 0; n < lz::kT0; ++n) hp->t0c[size_t(row) * lz::kT0 + n] = double(cf[n]);
        };
        for (int j = 0; j < hp->nctx; ++j)
            if (plain[j]->k.branch != lz::kTrivial) fill(plain[j]->k, j, 0);
        if (hess) {
            fill(hess->k, hp->nctx, 1);
            fill(hess->k, hp->nctx + 1, 2);
        }
        hp->n_t0 = std::min(need, lz::kT0);
        hp->t0_rho_max = ok ? double(rho_max) : -1.0;
        // the Hessian rows as pieces (line kernel): series evaluated in long double at the
        // Chebyshev nodes of each bin; kept only if every piece meets 1e-15 of the row's scale
        hp->q0tab.clear();
        hp->q0_nb = 0;
        if (hess && ok) {
            const int nb = int(std::ceil(double(c_l * rho_max / ld(lz::kBinWidth)) - 1e-12));
            const int ps = lz::piece_stride(2);
            std::vector<double> tab(size_t(nb) * ps, 0.0);
            bool fit_ok = nb > 0;
            for (int row = 0; row < 2 && fit_ok; ++row) {
                const double* cf = &hp->t0c[size_t(hp->nctx + row) * lz::kT0];
                auto g = [&](ld x) {
                    const ld r = x / c_l;
                    ld acc = 0.0L;
                    for (int n = lz::kT0 - 1; n >= 0; --n) acc = acc * r + ld(cf[n]);
                    return acc;
                };
                ld scale = 0.0L;
                for (int i = 0; i <= 8 * nb; ++i) scale = std::max(scale, std::fabs(g(ld(lz::kBinWidth) * i / 8.0L)));
                for (int b = 0; b < nb; ++b) {
                    double pc[lz::kNC];
                    const double err = lz::fit_piece_fn(g, ld(lz::kBinWidth) * b, ld(lz::kBinWidth) * (b + 1), pc);
                    if (err > 1e-15 * double(scale)) fit_ok = false;
                    for (int m = 0; m < 8; ++m) tab[size_t(b) * ps + row * 8 + m] = pc[m];
                    tab[size_t(b) * ps + 16 + row] = pc[8];
                }
            }
            if (fit_ok) {
                hp->q0tab.swap(tab);
                hp->q0_nb = nb;
                hp->q0_inv_h = double(c_l / ld(lz::kBinWidth));
            }
        }
    });
    // LATSUM_TIMING=1: host phase times of the plan build on stderr (tuning aid)
    const bool timing = std::getenv("LATSUM_TIMING") != nullptr;
    auto tprev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  plan %-18s %.3f ms\n", what, std::chrono::duration<double, std::milli>(now - tprev).count());
        tprev = now;
    };
    union_points(d, dsets, &hp->dir_n);
    std::vector<double> rec_n;
    union_points(d, rsets, &rec_n);
    lap("unions");
    // Ball truncation of the direct set: the reference appends whole max-norm shells
    // (L/epstein.py:134-149), i.e. a half cube whose corners carry weights many orders below
    // its 1e-18 term cutoff; points whose every channel is below `dcut` (default 1e-18) times
    // the summed weights are dropped (|z|^2 factor covers the Hessian channels).
    // weights of the direct-channel contexts at every union point for the ball truncation: the
    // contexts' own weights (the reference's double-precision w_z, L/epstein.py:139) where the
    // point is in that context's set, else the same formula; the kept points' channel weights are
    // then recomputed in long double.
    // Trace-Z plans carry only the Hessian channel, so only its weights matter there.
    std::vector<const lz::HostCtx*> wctx;
    if (!trace_z) wctx.assign(plain.begin(), plain.end());
    if (hess) wctx.push_back(hess);
    WeightMap wmap;
    wmap.nw = wctx.size();
    {
        ld dcut = trace_z ? ld(lz::kAtmTermCutoff) : 1e-18L;
        if (const char* e = std::getenv("LATSUM_DIRECT_CUTOFF")) dcut = std::strtold(e, nullptr);
        const size_t np = hp->dir_n.size() / d;
        // one context whose own set is the union (trace-Z plans): its weights align by index
        const std::vector<double>* aligned = nullptr;
        if (wctx.size() == 1 && dsets.size() == 1) {
            const bool h = wctx[0] == hess;
            if (dsets[0] == (h ? &hess->hdir_n : &wctx[0]->dir_n)) aligned = h ? &hess->hdir_w : &wctx[0]->dir_w;
        }
        std::vector<std::unordered_map<uint64_t, double>> known(aligned ? 0 : wctx.size());
        for (size_t j = 0; j < known.size(); ++j) {
            const bool h = wctx[j] == hess;
            const std::vector<double>& nn = h ? hess->hdir_n : wctx[j]->dir_n;
            const std::vector<double>& ww = h ? hess->hdir_w : wctx[j]->dir_w;
            known[j].reserve(ww.size() * 2);
            for (size_t i = 0; i < ww.size(); ++i) known[j].emplace(pack_key(d, &nn[i * d]), ww[i]);
        }
        lap("known maps");
        std::vector<double> wv(np * wctx.size()), mag(np, 0.0);
        lz::parallel_for(int64_t(np), 256, [&](int64_t i) {
            double r2 = 0.0;
            for (int a = 0; a < d; ++a) {
                double za = 0.0;
                for (int b = 0; b < d; ++b) za += first->A[a * d + b] * hp->dir_n[i * d + b];
                r2 += za * za;
            }
            if (aligned) {
                const double w = (*aligned)[size_t(i)];
                wv[i] = w;
                mag[i] = std::fabs(w) * std::max(1.0, r2);
                return;
            }
            const uint64_t key = pack_key(d, &hp->dir_n[i * d]);
            for (size_t j = 0; j < wctx.size(); ++j) {
                const auto it = known[j].find(key);
                double w;
                if (it != known[j].end()) {
                    w = it->second;
                } else {
                    const double nu = wctx[j]->k.nu;
                    w = lz::upper_gamma<double>(nu / 2.0, lz::kPi * wctx[j]->k.split * r2) * std::pow(r2, -nu / 2.0);
                }
                wv[i * wctx.size() + j] = w;
                mag[i] = std::max(mag[i], std::fabs(w) * std::max(1.0, r2));
            }
        });
        double total = 0.0;  // fixed summation order: independent of the thread count
        for (double w : wv) total += std::fabs(w);
        std::vector<double> kept;
        for (size_t i = 0; i < np; ++i)
            if (mag[i] > double(dcut) * total)
                kept.insert(kept.end(), hp->dir_n.begin() + i * d, hp->dir_n.begin() + (i + 1) * d);
        // the kept points' weights in long double: the double-precision w_z are good to ~1e-15,
        // which the cancellation between the regular and singular parts near the log-case
        // exponents (nu -> d + 2m) can amplify past the 1e-12 parity bar
        const size_t nk = kept.size() / d, nwc = wctx.size();
        wmap.rows.assign(nk * nwc, 0.0L);
        // w_z depends on |z|^2 only: points on one shell of the lattice's symmetry (fcc at the ATM
        // split: 6,107 points, ~140 distinct radii) share one evaluation: the group's first point
        // is evaluated (members equal it within 64 long-double roundings of the three-term sum of
        // squares -- far below the weight's sensitivity).
        std::vector<ld> r2v(nk);
        for (size_t i = 0; i < nk; ++i) {
            ld r2 = 0.0L;
            for (int a = 0; a < d; ++a) {
                ld za = 0.0L;
                for (int b = 0; b < d; ++b) za += ld(first->A[a * d + b]) * kept[i * d + b];
                r2 += za * za;
            }
            r2v[i] = r2;
        }
        // groups by the double rounding of |z|^2 (hash), members checked against the group's
        // long-double value (a point that does not match opens its own group)
        std::vector<uint32_t> rep, group(nk);  // rep: first point of every group
        {
            std::unordered_map<uint64_t, uint32_t> seen;
            seen.reserve(nk / 4 + 16);
            for (size_t i = 0; i < nk; ++i) {
                const double r2d = double(r2v[i]);
                uint64_t bits;
                std::memcpy(&bits, &r2d, sizeof(bits));
                const auto it = seen.emplace(bits, uint32_t(rep.size()));
                if (!it.second && std::fabs(r2v[i] - r2v[rep[it.first->second]]) <= 64.0L * LDBL_EPSILON * r2v[i]) {
                    group[i] = it.first->second;
                } else {
                    group[i] = uint32_t(rep.size());
                    rep.push_back(uint32_t(i));
                }
            }
        }
        std::vector<ld> gw(rep.size() * nwc);
        lz::parallel_for(int64_t(rep.size()), 8, [&](int64_t gi) {
            ld z[lz::kMaxDim];
            for (size_t j = 0; j < nwc; ++j) gw[size_t(gi) * nwc + j] = direct_weight(*wctx[j], &kept[size_t(rep[gi]) * d], z);
        });
        for (size_t i = 0; i < nk; ++i)
            for (size_t j = 0; j < nwc; ++j) wmap.rows[i * nwc + j] = gw[size_t(group[i]) * nwc + j];
        wmap.keys.resize(nk);
        for (size_t i = 0; i < nk; ++i) wmap.keys[i] = pack_key(d, &kept[i * d]);
        hp->dir_n.swap(kept);
    }
    lap("union+ball");
    // Direct points as 2D slabs: slab = fixed (n_1 .. n_{d-2}), rows along n_{d-1}, columns along
    // n_d.  The kernel evaluates one sincos per slab; row starts follow by a complex rotation
    // exp(2 pi i kappa_{d-1}) and points along a row by the Chebyshev cosine recurrence in
    // kappa_d.  Rows are stored from their first point (skip = columns after the slab's l0),
    // padded to even length with zero weights (the kernel walks rows two points at a time).
    // Hessian: the direct term -8 pi^2 w z_a z_b cos(.) is stored divided by 4 rfac so that it
    // shares the kernel's reciprocal accumulators (sum of y_a y_b F''), and factorised over the
    // slab: z = zc + j' e2 + l' e3 (zc = slab center, e2 = A e_{d-1}, e3 = A e_d), so three
    // channels w l'^m (m = 0, 1, 2) replace the d(d+1)/2 channels w z_a z_b and the row and
    // slab folds carry the j' and zc parts.
    // ATM kernel form (LATSUM_LINE): 2 (default) row-factorised direct block, 1 line block staged
    // in shared memory, 0 slab walk
    int line_env = 2;
    if (const char* e = std::getenv("LATSUM_LINE")) line_env = std::atoi(e);
    const ld hscale = hess ? -2.0L * ld(lz::kPi) * ld(lz::kPi) / ld(hess->k.rfac) : 0.0L;
    const int hw = int(wctx.size()) - 1;  // the Hessian context's slot in the wmap rows
    hp->line.clear();
    hp->row_on = 0;
    {
        const size_t np = hp->dir_n.size() / d;
        // lexicographic order = order of the packed keys (most significant field first; the
        // points are distinct, so no ties).  The sort works on copies, so the row-factorised block
        // (which groups the points itself and takes them in any order) is built beside it.
        std::vector<double> pts(np * d);
        std::vector<uint32_t> sorted_row(np);
        std::vector<int> runs;
        auto sort_job = [&]() {
            std::vector<std::pair<uint64_t, uint32_t>> ord(np);
            for (size_t i = 0; i < np; ++i) ord[i] = {wmap.keys[i], uint32_t(i)};
            std::sort(ord.begin(), ord.end());
            for (size_t i = 0; i < np; ++i) {
                for (int a = 0; a < d; ++a) pts[i * d + a] = hp->dir_n[size_t(ord[i].second) * d + a];
                sorted_row[i] = ord[i].second;
            }
            auto key = [&](size_t i, int a) { return std::lround(pts[i * d + a]); };
            // maximal runs (for plan info only)
            for (size_t i = 0; i < np; ++i) {
                bool cont = i > 0;
                for (int a = 0; cont && a < d - 1; ++a) cont = key(i, a) == key(i - 1, a);
                cont = cont && key(i, d - 1) == key(i - 1, d - 1) + 1;
                if (cont) {
                    runs.back() += 1;
                } else {
                    runs.push_back(int(i));
                    runs.push_back(1);
                }
            }
        };
        if (trace_z && d == 3 && line_env >= 2 && hess) {
            std::future<void> sj = std::async(std::launch::async, sort_job);
            wmap.row_of.resize(np);
            for (size_t i = 0; i < np; ++i) wmap.row_of[i] = uint32_t(i);  // rows follow the unsorted order
            build_row_block(hp, wmap, first->A, hscale, hw);
            sj.get();
        } else {
            sort_job();
        }
        hp->dir_n.swap(pts);
        wmap.row_of.swap(sorted_row);
        hp->run_info.swap(runs);
    }
    const int nh = hess ? 3 : 0;
    if (trace_z && !hess) throw Error{LZ_EINVAL, "trace-Z plans need the Hessian context"};
    hp->dir_plain = trace_z ? 0 : hp->nctx;
    hp->nw = trace_z ? nh : ((hp->nctx + nh == 1) ? 1 : ((hp->nctx + nh + 1) & ~1));
    for (int a = 0; a < 4; ++a) hp->e2[a] = hp->e3[a] = 0.0;
    for (int a = 0; a < d; ++a) {
        hp->e3[a] = first->A[a * d + d - 1];
        if (d >= 2) hp->e2[a] = first->A[a * d + d - 2];
    }
    // the slab block (built last, below, unless the line block replaces it)
    auto build_slab = [&]() {
    {
        const size_t np = hp->dir_n.size() / d;
        const int ns = std::max(d - 2, 0);   // slab key length
        struct Row { long j; std::vector<std::pair<long, size_t>> pts; };
        std::vector<std::pair<std::vector<long>, std::vector<Row>>> slabs;
        for (size_t i = 0; i < np; ++i) {
            const double* n = &hp->dir_n[i * d];
            std::vector<long> sk(ns);
            for (int a = 0; a < ns; ++a) sk[a] = std::lround(n[a]);
            const long j = d >= 2 ? std::lround(n[d - 2]) : 0;
            const long l = std::lround(n[d - 1]);
            if (slabs.empty() || slabs.back().first != sk) slabs.push_back({sk, {}});
            auto& rows = slabs.back().second;
            if (rows.empty() || rows.back().j != j) rows.push_back({j, {}});
            rows.back().pts.push_back({l, i});
        }
        const int sr = 2 * d + 2;
        std::vector<double> srec, rrec, wts_out;
        int n_rows = 0;
        for (const auto& sl : slabs) {
            const auto& rows = sl.second;
            const long jmin = rows.front().j, jmax = rows.back().j;
            long l0 = rows.front().pts.front().first, l1 = l0;
            for (const Row& r : rows) {
                l0 = std::min(l0, r.pts.front().first);
                l1 = std::max(l1, r.pts.back().first);
            }
            const ld jc = ld(jmin + jmax) / 2.0L, lc = ld(l0 + l1) / 2.0L;
            std::vector<double> rec(sr, 0.0);
            ld ncen[lz::kMaxDim];
            for (int a = 0; a < ns; ++a) {
                rec[a] = double(sl.first[a]);
                ncen[a] = ld(sl.first[a]);
            }
            if (d >= 2) {
                rec[d - 2] = double(jmin);
                ncen[d - 2] = jc;
            }
            rec[d - 1] = double(l0);
            ncen[d - 1] = lc;
            for (int a = 0; a < d; ++a) {
                ld zc = 0.0L;
                for (int b = 0; b < d; ++b) zc += ld(first->A[a * d + b]) * ncen[b];
                rec[d + a] = double(zc);
            }
            rec[2 * d] = double(ld(jmin) - jc);
            const int32_t sinfo[2] = {n_rows, int32_t(jmax - jmin + 1)};
            std::memcpy(&rec[2 * d + 1], sinfo, sizeof(sinfo));
            srec.insert(srec.end(), rec.begin(), rec.end());
            size_t ri = 0;
            for (long j = jmin; j <= jmax; ++j, ++n_rows) {
                int32_t rinfo[2] = {0, 0};
                if (ri < rows.size() && rows[ri].j == j) {
                    const Row& r = rows[ri++];
                    const long lo = r.pts.front().first, hi = r.pts.back().first;
                    // rows padded to even length (16-byte pairs of points), to a multiple of 4
                    // for one-channel plans (the kernel's plain-zeta row loop takes 4 points per step)
                    const long len = hi - lo + 1, skip = lo - l0;
                    const long lenp = hp->nw == 1 ? (len + 3) & ~3L : len + (len & 1);
                    if (lenp > 65535 || skip > 65535) throw Error{LZ_EINVAL, "direct row too long"};
                    const size_t row0 = wts_out.size() / hp->nw;
                    if (row0 > size_t(INT32_MAX)) throw Error{LZ_EINVAL, "direct set too large"};
                    rinfo[0] = int32_t(row0);
                    rinfo[1] = int32_t((skip << 16) | lenp);
                    wts_out.resize(wts_out.size() + size_t(lenp) * hp->nw, 0.0);
                    for (const auto& pt : r.pts) {
                        const size_t base = (row0 + size_t(pt.first - lo)) * hp->nw;
                        const ld* w = wmap.at(pack_key(d, &hp->dir_n[pt.second * d]));
                        const int dp = hp->dir_plain;
                        for (int c = 0; c < dp; ++c) wts_out[base + c] = double(w[c]);
                        if (hess) {
                            const ld wh = w[hw] * hscale, lp = ld(pt.first) - lc;
                            wts_out[base + dp] = double(wh);
                            wts_out[base + dp + 1] = double(wh * lp);
                            wts_out[base + dp + 2] = double(wh * lp * lp);
                        }
                    }
                }
                double rd;
                std::memcpy(&rd, rinfo, sizeof(rd));
                rrec.push_back(rd);
            }
        }
        hp->n_slabs = int(slabs.size());
        hp->n_rows = n_rows;
        if (rrec.size() & 1) rrec.push_back(0.0);
        hp->direct = srec;
        hp->rows_off = int(srec.size());
        hp->direct.insert(hp->direct.end(), rrec.begin(), rrec.end());
        hp->w_off = int(hp->direct.size());
        hp->direct.insert(hp->direct.end(), wts_out.begin(), wts_out.end());
        hp->n_wrows = int(wts_out.size() / hp->nw);
    }
    };
    lap("sort");
    // (the row-factorised block was built beside the sort, above)
    if (trace_z && d == 3 && !hp->row_on && line_env >= 1 && !build_line_block(hp, wmap, first->A, hscale, hw))
        hp->line.clear();
    lap("line block");
    // reciprocal points, sorted by |q| (stable) for the per-warp culling bound
    const size_t nrec = rec_n.size() / d;
    std::vector<double> q(nrec * d);
    std::vector<ld> qn(nrec);
    for (size_t i = 0; i < nrec; ++i) {
        ld r2 = 0.0L;
        for (int a = 0; a < d; ++a) {
            ld v = 0.0L;
            for (int b = 0; b < d; ++b) v += ld(first->B[a * d + b]) * rec_n[i * d + b];
            q[i * d + a] = double(v);
            r2 += v * v;
        }
        qn[i] = std::sqrt(r2);
    }
    std::vector<size_t> order(nrec);
    for (size_t i = 0; i < nrec; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return qn[a] < qn[b]; });
    hp->rec_q.assign(nrec * d, 0.0);
    hp->rec_norm.assign(nrec, 0.0);
    for (size_t i = 0; i < nrec; ++i) {
        for (int a = 0; a < d; ++a) hp->rec_q[i * d + a] = q[order[i] * d + a];
        hp->rec_norm[i] = double(qn[order[i]]);
    }
    {
        const int qs = (d + 1) & ~1;
        hp->rq_pad.assign(nrec * qs, 0.0);
        for (size_t i = 0; i < nrec; ++i)
            for (int a = 0; a < d; ++a) hp->rq_pad[i * qs + a] = hp->rec_q[i * d + a];
    }
    lap("reciprocal sort");
    q0_job.get();  // q = 0 series and pieces (started with the table fit)
    lap("q=0 series");
    if (!table_job.valid()) {
        hp->tab = lz::HostTable();
        hp->tab.nfunc = nf;
    } else {
        table_job.get();
        // beyond x_hi every tabulated function is exactly zero in the kernel
        hp->r_cut = double(std::sqrt(ld(hp->tab.x_hi) / c) * (1.0L + 1e-9L));
        hp->r_in = double(std::sqrt(ld(hp->tab.x_hi) / c) * (1.0L - 1e-9L));
    }
    lap("table wait");
    // The line kernel (kernels.cu tile_kernel_l) does not read the slab block: skip it when the
    // line block exists, the kernel is not disabled (LATSUM_LINE=0) and its shared-memory image
    // (everything but the slab block, the count table and 24 warp scratches) fits comfortably.
    bool need_slab = hp->line.empty() && !hp->row_on;
    if (!need_slab) {
        const size_t qs = size_t((d + 1) & ~1);
        auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
        const size_t img = a16(8 * hp->rec_norm.size() * qs) + a16(8 * hp->rec_norm.size()) +
                           a16(8 * hp->tab.coef.size()) + a16(4 * hp->tab.dir.size()) +
                           a16(8 * size_t(hp->nctx + 2) * lz::kT0) + a16(hp->line.size());
        // (row kernel: 20 warps x kRowScrBytes, the q = 0 pieces, the count table, angular nodes)
        const size_t extra = hp->row_on ? 20 * 7120 + 13 * 1024 : 1024 + 24 * 4000 + 8192;
        need_slab = line_env == 0 || img + extra > 227 * 1024 ||
                    hp->rec_norm.size() > 512 ||  // kernels.cu kLineQ
                    hp->q0_nb < 1 || hp->q0_nb > 48;  // kernels.cu kQ0Max
        if (need_slab) hp->row_on = 0;
    }
    if (need_slab) build_slab();
    lap("slab block");
}

// All device arrays of a plan in one allocation and one copy (16-byte aligned sections).
struct Blob {
    std::vector<unsigned char> host;
    template <class T> size_t add(const T* p, size_t n) {
        const size_t off = (host.size() + 15) & ~size_t(15);
        host.resize(off + n * sizeof(T));
        if (n) std::memcpy(host.data() + off, p, n * sizeof(T));
        return off;
    }
};

lz::DevPlan upload_plan(const HostPlan& hp, std::vector<void*>* allocs) {
    lz::DevPlan P;
    std::memset(&P, 0, sizeof(P));
    // reciprocal vectors padded to an even stride (16-byte aligned double2 loads)
    const std::vector<double>& rq = hp.rq_pad;
    // section order and 16-byte alignment = the kernel's shared-memory image (stage<true>), so the
    // kernel stages the plan with one bulk copy
    Blob b;
    const size_t o_dir = b.add(hp.direct.data(), hp.direct.size());
    const size_t o_rq = b.add(rq.data(), rq.size());
    const size_t o_rn = b.add(hp.rec_norm.data(), hp.rec_norm.size());
    const size_t o_cf = b.add(hp.tab.coef.data(), hp.tab.coef.size());
    const size_t o_td = b.add(hp.tab.dir.data(), hp.tab.dir.size());
    std::vector<double> t0rows(size_t(hp.nctx + (hp.hess ? 2 : 0)) * lz::kT0, 0.0);
    std::copy(hp.t0c.begin(), hp.t0c.begin() + std::min(hp.t0c.size(), t0rows.size()), t0rows.begin());
    const size_t o_t0 = b.add(t0rows.data(), t0rows.size());
    if (!hp.line.empty()) b.add(hp.line.data(), hp.line.size());  // last section (kernels.cu stage)
    b.host.resize((b.host.size() + 15) & ~size_t(15), 0);
    unsigned char* dev = nullptr;
    if (!b.host.empty()) {
        check_cuda(cudaMalloc(reinterpret_cast<void**>(&dev), b.host.size()), "cudaMalloc");
        allocs->push_back(dev);
        copy_h2d(dev, b.host.data(), b.host.size(), nullptr, false);
    }
    auto at = [&](size_t off, bool nonempty) -> unsigned char* { return nonempty ? dev + off : nullptr; };
    P.blob = dev;
    P.blob_bytes = b.host.size();
    P.d = hp.d;
    P.nctx = hp.nctx;
    P.hess = hp.hess;
    P.n_dir = hp.n_wrows;  // padded weight rows
    P.n_rec = int(hp.rec_q.size() / hp.d);
    P.nw = hp.nw;
    P.c = hp.c;
    P.alias_fp = hp.alias_fp;
    P.t0c = reinterpret_cast<const double*>(at(o_t0, !t0rows.empty()));
    P.n_t0 = hp.n_t0;
    P.t0_rho_max = hp.t0_rho_max;
    P.alias_ratio = hp.alias_ratio;
    std::memcpy(P.A, hp.A, sizeof(P.A));
    std::memcpy(P.B, hp.B, sizeof(P.B));
    P.direct = reinterpret_cast<const double*>(at(o_dir, !hp.direct.empty()));
    P.direct_host = hp.direct.empty() ? nullptr : hp.direct.data();
    P.n_direct = int(hp.direct.size());
    P.t0_host = hp.t0c.data();
    P.rq_host = hp.rq_pad.data();
    P.q0_host = hp.q0tab.data();
    P.q0_nb = hp.q0_nb;
    P.q0_inv_h = hp.q0_inv_h;
    if (hp.hess) {
        const lz::CtxConst& k = hp.hctx;
        P.h_kk = k.sing_coef * k.inv_vol / (k.pref * k.rfac);
        P.h_cm = -4.0 * k.pref * k.rfac / (4.0 * lz::kPi * lz::kPi);
    }
    P.line_bytes = unsigned(hp.line.size());
    P.line_sign = hp.line_sign;
    P.row_on = hp.row_on;
    P.row_nJ = hp.row_nJ;
    P.row_PS = hp.row_PS;
    P.row_NI = hp.row_NI;
    for (int a = 0; a < 3; ++a) P.row_jmin[a] = hp.row_jmin[a];
    P.row_cand_max = 64;  // kernels.cu kRowCand
    if (const char* e = std::getenv("LATSUM_ROW_CAND_MAX")) P.row_cand_max = std::max(0, std::min(64, std::atoi(e)));
    if (hp.row_on) {
        P.row_pts = upload(hp.row_pts, allocs);
        P.row_idx = upload(hp.row_idx, allocs);
    }
    for (int a = 0; a < 3; ++a) {
        P.line_K[a] = hp.line_K[a];
        P.line_P[a] = hp.line_P[a];
        P.line_slot_off[a] = hp.line_slot_off[a];
        P.line_meta_off[a] = hp.line_meta_off[a];
    }
    P.n_slabs = hp.n_slabs;
    P.n_rows = hp.n_rows;
    P.rows_off = hp.rows_off;
    P.w_off = hp.w_off;
    std::memcpy(P.e2, hp.e2, sizeof(P.e2));
    std::memcpy(P.e3, hp.e3, sizeof(P.e3));
    P.rec_q = reinterpret_cast<const double*>(at(o_rq, !rq.empty()));
    P.rec_norm = reinterpret_cast<const double*>(at(o_rn, !hp.rec_norm.empty()));
    P.r_cut = hp.r_cut;
    P.r_in = hp.r_in;
    P.tab.dir = reinterpret_cast<const int*>(at(o_td, !hp.tab.dir.empty()));
    P.tab.coef = reinterpret_cast<const double*>(at(o_cf, !hp.tab.coef.empty()));
    P.tab.nbins = hp.tab.nbins;
    P.tab.nfunc = hp.tab.nfunc;
    P.tab.npieces = hp.tab.npieces;
    P.tab.ncoef = int(hp.tab.coef.size());
    P.tab.x_lo = hp.tab.x_lo;
    P.tab.inv_hb = hp.tab.inv_hb;
    P.tab.x_hi = hp.tab.x_hi;
    P.tab.c = hp.c;
    P.tab.r_scale = hp.c * hp.tab.inv_hb;
    P.tab.x_off = hp.tab.x_lo * hp.tab.inv_hb;
    P.tab.xb_max = double(hp.tab.nbins) - 1.0 / 1048576.0;
    P.tab.r_off = hp.c > 0.0 ? double((long double)hp.tab.x_lo / (long double)hp.c) : 0.0;
    P.tab.nbins_d = double(hp.tab.nbins);
    // radius of the first low-degree bin's left edge (x_switch = x_lo + lo_start h, rho = x / c)
    P.tab.r_lo = (hp.tab.lo_start < hp.tab.nbins && hp.c > 0.0)
                     ? double(std::sqrt((ld(hp.tab.x_lo) + ld(hp.tab.lo_start) / ld(hp.tab.inv_hb)) / ld(hp.c)))
                     : 0.0;
    // branch-free lookup is opt-in (LATSUM_BRANCHFREE=1): measured slower on the fcc ATM grid,
    // where warps beyond the cutoff otherwise skip the polynomial entirely
    const char* bf = std::getenv("LATSUM_BRANCHFREE");
    P.tab.branchfree = (bf && std::atoi(bf) == 1) ? 1 : 0;
    P.tab.has_marker = 0;
    for (int e : hp.tab.dir)
        if ((e & 15) == lz::kDirectMarker) P.tab.has_marker = 1;
    if (hp.tab.nbins == 0) P.tab.has_marker = 1;  // no table: never evaluated (no q points)
    for (int j = 0; j < 4; ++j) {
        P.tab.p[j] = hp.tab.p[j];
        P.tab.scale[j] = hp.tab.scale[j];
    }
    for (int j = 0; j < lz::kMaxCtx; ++j) P.ctx[j] = hp.ctx[j];
    P.hctx = hp.hctx;
    return P;
}

struct GridArrays {
    double* u = nullptr;
    double* wu = nullptr;
    double* v = nullptr;
    double* wv = nullptr;
};

// Per-device scratch for the host-buffer entry points: one non-blocking stream,
// grow-only device memory and grow-only pinned staging, reused across calls so a
// call costs copies + kernels only (no allocation, no stream creation).
struct Arena {
    std::mutex mu;
    cudaStream_t st = nullptr;
    char* dbuf = nullptr;
    size_t dcap = 0;
    char* hbuf = nullptr;
    size_t hcap = 0;
    void ensure(size_t dbytes, size_t hbytes) {
        if (!st) check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        if (dbytes > dcap) {
            if (dbuf) cudaFree(dbuf);
            dcap = std::max(dbytes, dcap * 2);
            check_cuda(cudaMalloc((void**)&dbuf, dcap), "arena malloc");
        }
        if (hbytes > hcap) {
            if (hbuf) cudaFreeHost(hbuf);
            hcap = std::max(hbytes, hcap * 2);
            check_cuda(cudaHostAlloc((void**)&hbuf, hcap, cudaHostAllocDefault), "arena pinned alloc");
        }
    }
};

std::mutex g_arena_mu;
std::map<int, Arena*> g_arenas;

Arena& arena(int device) {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    Arena*& a = g_arenas[device];
    if (!a) a = new Arena();
    return *a;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

// H2D from a host buffer: direct DMA when pinned, else through the arena's pinned staging.
void h2d(void* dst, const void* src, size_t bytes, char* staging, cudaStream_t st) {
    if (bytes == 0) return;
    if (is_pinned(src)) {
        copy_h2d(dst, src, bytes, st);
    } else {
        std::memcpy(staging, src, bytes);
        copy_h2d(dst, staging, bytes, st);
    }
}

}  // namespace

struct lz_ctx {
    lz::HostCtx h;
    int device = -1;
    // evaluation tables are built on first use (plans of fused kernels build their own)
    std::mutex mu;
    bool plain_ready = false, hess_ready = false, big_ready = false;
    HostPlan plain, hessp, plain_big;
    lz::DevPlan dplain, dhess, dplain_big;
    std::vector<void*> allocs;
    // order-m derivative plans (deriv.cu), built on first use
    std::map<int, lz::DevDeriv> dderiv;
    std::map<int, lz::HostTable> dtab;
    // moment-form plans keyed by (order, taylor, point-set order)
    std::map<std::tuple<int, int, int>, lz::DevDeriv> dderiv_g;
    std::map<std::tuple<int, int, int>, lz::HostTable> dtab_g;
};

struct lz_plan {
    int device = -1;
    int kind = 0;  // 0 product, 1 atm
    int d = 0;
    int mult[4] = {0, 0, 0, 0};
    HostPlan hp;
    lz::DevPlan P;
    std::vector<void*> allocs;
    mutable std::mutex mu;
};

namespace {

void fill_grid(int d, const lz_grid* g, lz::DevGrid* dg) {
    if (g->n_u < 1 || (d > 1 && g->n_v < 1) || g->grading < 1)
        throw Error{LZ_EINVAL, "grid sizes must be positive and grading >= 1"};
    if (!(g->u_lo >= 0.0 && g->u_lo < 0.5)) throw Error{LZ_EINVAL, "u_lo must lie in [0, 1/2)"};
    dg->n_u = g->n_u;
    dg->n_v = d > 1 ? g->n_v : 1;
    dg->n_cell = (1 << (d - 1)) * d;
    // warp patch: pu radial x pv angular nodes (pu * pv = 32); compact patches keep the
    // per-warp culling radius and the table pieces of the 32 lanes close together
    int pu = 1;  // measured best on B200 for the fcc ATM grid
    if (const char* e = std::getenv("LATSUM_PATCH_U")) pu = std::atoi(e);
    if (pu != 1 && pu != 2 && pu != 4 && pu != 8 && pu != 16 && pu != 32) pu = 1;
    dg->pu = d > 1 ? pu : 32;
    dg->pv = d > 1 ? 32 / pu : 1;
    dg->npu = (dg->n_u + dg->pu - 1) / dg->pu;
    dg->npv = d > 1 ? (dg->n_v + dg->pv - 1) / dg->pv : 1;
    dg->nv2 = d > 2 ? dg->n_v : 1;
    dg->n_patch = int64_t(dg->n_cell) * dg->nv2 * dg->npv * dg->npu;
    const int64_t n_tiles = (dg->n_patch + 7) / 8;
    dg->tile_lo = std::max<int64_t>(0, g->tile_lo);
    dg->tile_hi = g->tile_hi > 0 ? std::min(g->tile_hi, n_tiles) : n_tiles;
}

// Quadrature node arrays on the device, cached process-wide per (device, d, n_u, n_v, grading,
// u_lo): read-only and shared by every plan, so a cold plan does not re-upload them.
std::mutex g_grid_mu;
std::map<std::tuple<int, int, int, int, int, double>, GridArrays> g_grid_cache;

const GridArrays& grid_arrays(const lz_plan* plan, const lz_grid* g) {
    auto& cache = g_grid_cache;
    const int d = plan->d;
    std::lock_guard<std::mutex> lock(g_grid_mu);
    auto key = std::make_tuple(plan->device, d, g->n_u, d > 1 ? g->n_v : 1, g->grading, g->u_lo);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<double> x, w;
    lz::gauss_legendre(g->n_u, &x, &w);
    std::vector<double> u(g->n_u), wu(g->n_u);
    const ld q = g->grading, ulo = g->u_lo, span = 0.5L - ld(g->u_lo);
    for (int i = 0; i < g->n_u; ++i) {
        // t = (x+1)/2 on (0,1); u = u_lo + (1/2 - u_lo) t^q; du = (1/2 - u_lo) q t^{q-1} dt; times u^{d-1}
        const ld t = (ld(x[i]) + 1.0L) / 2.0L;
        const ld wt = ld(w[i]) / 2.0L;
        const ld uu = ulo + span * std::pow(t, q);
        u[i] = double(uu);
        wu[i] = double(wt * span * q * std::pow(t, q - 1.0L) * std::pow(uu, ld(d - 1)));
    }
    std::vector<double> v, wv;
    if (d > 1) {
        lz::gauss_legendre(g->n_v, &x, &w);
        v.resize(g->n_v);
        wv.resize(g->n_v);
        // angular_nodes: v = (x + 1)/4, weights w/4 (L/quadrature.py:165-177)
        for (int i = 0; i < g->n_v; ++i) {
            v[i] = double((ld(x[i]) + 1.0L) / 4.0L);
            wv[i] = double(ld(w[i]) / 4.0L);
        }
    } else {
        v.assign(1, 0.0);
        wv.assign(1, 1.0);
    }
    GridArrays ga;
    std::vector<void*> allocs;  // process lifetime
    std::vector<double> all;
    all.reserve(2 * (u.size() + v.size()));
    all.insert(all.end(), u.begin(), u.end());
    all.insert(all.end(), wu.begin(), wu.end());
    all.insert(all.end(), v.begin(), v.end());
    all.insert(all.end(), wv.begin(), wv.end());
    double* dev = upload(all, &allocs);  // one allocation, one copy
    ga.u = dev;
    ga.wu = dev + u.size();
    ga.v = dev + 2 * u.size();
    ga.wv = dev + 2 * u.size() + v.size();
    return cache.emplace(key, ga).first->second;
}

// Tile-kernel scratch (warp partials + per-tile arrival counters) per (device, stream): kernels on
// one stream are serialised, so they can share it; grown stream-ordered (cudaMallocAsync /
// cudaFreeAsync from the device's memory pool), counters zeroed on growth and left zero by every
// completed launch.
struct Scratch {
    double* wpart = nullptr;        // [cap_w * 8][2] warp partials (only launches that need them)
    unsigned int* tcount = nullptr; // [cap + 2]: tile counters, then the work-queue counters
    double* dtab = nullptr;         // row-factorised ATM kernel: D table (grow-only)
    int64_t cap = 0, cap_w = 0;
    size_t cap_d = 0;               // bytes

};
std::mutex g_scratch_mu;
std::map<std::pair<int, cudaStream_t>, Scratch> g_scratch;

// The device's default memory pool keeps freed memory (release threshold: unlimited), so a
// scratch re-allocation after lz_release_caches does not map new pages at every cold call.
void keep_pool(int device) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (!done.insert(device).second) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}

void tile_scratch(int device, cudaStream_t st, int64_t n_tiles, bool need_wpart, double** wpart,
                  unsigned int** tcount, unsigned int** work, size_t dtab_bytes = 0, double** dtab = nullptr) {
    keep_pool(device);
    auto& pool = g_scratch;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    Scratch& s = pool[std::make_pair(device, st)];
    if (s.cap < n_tiles) {
        if (s.tcount) check_cuda(cudaFreeAsync(s.tcount, st), "cudaFreeAsync");
        const size_t cbytes = (size_t(n_tiles) + 2) * sizeof(unsigned int);
        void* p = nullptr;
        check_cuda(cudaMallocAsync(&p, cbytes, st), "cudaMallocAsync");
        s.tcount = static_cast<unsigned int*>(p);
        check_cuda(cudaMemsetAsync(s.tcount, 0, cbytes, st), "cudaMemsetAsync");
        s.cap = n_tiles;
    }
    if (need_wpart && s.cap_w < n_tiles) {
        if (s.wpart) check_cuda(cudaFreeAsync(s.wpart, st), "cudaFreeAsync");
        void* p = nullptr;
        check_cuda(cudaMallocAsync(&p, size_t(n_tiles) * 8 * 2 * sizeof(double), st), "cudaMallocAsync");
        s.wpart = static_cast<double*>(p);
        s.cap_w = n_tiles;
    }
    if (dtab_bytes > s.cap_d) {
        if (s.dtab) check_cuda(cudaFreeAsync(s.dtab, st), "cudaFreeAsync");
        void* p = nullptr;
        check_cuda(cudaMallocAsync(&p, dtab_bytes, st), "cudaMallocAsync");
        s.dtab = static_cast<double*>(p);
        s.cap_d = dtab_bytes;
    }
    if (dtab) *dtab = dtab_bytes ? s.dtab : nullptr;

    *wpart = need_wpart ? s.wpart : nullptr;
    *tcount = s.tcount;
    *work = s.tcount + s.cap;
}

// Lanes per point for the batch kernel: the smallest power of two that gives ~192 lanes per SM
// (C1 4096 points, graph-replay device time: G = 1 13.6 us, 4 10.2, 8 9.2, 16 9.5, 32 12.8;
// every lane repeats the per-node set-up, so more lanes than that cost more than they save).
int auto_lanes(int64_t n) {
    const int64_t target = 148LL * 192LL;
    int g = 1;
    while (g < 32 && n * g < target) g <<= 1;
    return g;
}

template <class F> int guarded(F&& f) {
    try {
        f();
        return LZ_OK;
    } catch (const Error& e) {
        return set_err(e.code, e.msg);
    } catch (const std::exception& e) {
        return set_err(LZ_EINVAL, e.what());
    }
}

}  // namespace

extern "C" {

const char* lz_version(void) { return "latsum_b200 0.1.0 (sm_100a, FP64)"; }

const char* lz_strerror(int code) {
    switch (code) {
        case LZ_OK: return "ok";
        case LZ_EINVAL: return "invalid argument";
        case LZ_EPOLE: return "pole of the meromorphic continuation";
        case LZ_ENONFINITE: return "k contains non-finite entries";
        case LZ_ECUDA: return "CUDA failure or no CUDA device";
        case LZ_ENCCL: return "collective failure";
        case LZ_ESHELLS: return "lattice sum did not truncate within shell budget";
        case LZ_ELATTICE: return "invalid lattice";
        case LZ_ESINGULAR: return "singular part undefined at k = 0";
    }
    return "unknown error";
}

const char* lz_last_error(void) { return g_last_error.c_str(); }

int lz_device_count(int* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *n = c;
    return LZ_OK;
}

namespace {

// Theta split of the per-context evaluation tables (zeta and Hessian batches), as a multiple
// of the context's own split (LATSUM_ZETA_SPLIT_SCALE, default 0.4: measured on B200, C1 2^20
// points 0.311 -> 0.170 ms).  Z is split-invariant; the context keeps reporting the
// reference's split and point sets (L/epstein.py:107).
double zeta_split_scale() {
    static double v = [] {
        const char* e = std::getenv("LATSUM_ZETA_SPLIT_SCALE");
        double x = e ? std::atof(e) : 0.4;
        return (x > 0.0 && x < 10.0) ? x : 0.4;
    }();
    return v;
}

// Large batches (>= kBigBatch points, G = 1: the kernel is shared-memory bound on the scattered
// table-piece loads) use a second plan at a smaller evaluation split, which moves terms from the
// table lookups to the broadcast direct-space loads (C1 2^20 points: 0.134 -> 0.119 ms; 4096
// points stay on the 0.4 plan: 8.4 vs 9.6 us).  LATSUM_ZETA_SPLIT_SCALE_BIG overrides 0.15.
constexpr int64_t kBigBatch = 65536;
double zeta_split_scale_big() {
    static double v = [] {
        const char* e = std::getenv("LATSUM_ZETA_SPLIT_SCALE_BIG");
        double x = e ? std::atof(e) : 0.15;
        return (x > 0.0 && x < 10.0) ? x : 0.15;
    }();
    return v;
}

void ensure_plain(const lz_ctx* cc) {
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    std::lock_guard<std::mutex> lock(c->mu);
    if (c->plain_ready) return;
    if (c->h.k.branch != lz::kTrivial) {
        const double sc = zeta_split_scale();
        if (sc != 1.0) {
            lz::HostCtx eval;
            lz::build_context(c->h.d, c->h.A, c->h.k.nu, c->h.k.split * sc, 0, &eval);
            build_host_plan({&eval}, nullptr, &c->plain);
        } else {
            build_host_plan({&c->h}, nullptr, &c->plain);
        }
    } else {
        c->plain.d = c->h.d;
        c->plain.nctx = 1;
        c->plain.ctx[0] = c->h.k;
        std::memcpy(c->plain.A, c->h.A, sizeof(c->plain.A));
        std::memcpy(c->plain.B, c->h.B, sizeof(c->plain.B));
    }
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        c->dplain = upload_plan(c->plain, &c->allocs);
    }
    c->plain_ready = true;
}

// the plain-zeta plan for a batch of n points (kBigBatch: the small-split plan)
const lz::DevPlan& plain_plan_for(const lz_ctx* cc, int64_t n) {
    ensure_plain(cc);
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    if (n < kBigBatch || c->h.k.branch == lz::kTrivial || zeta_split_scale_big() == zeta_split_scale())
        return c->dplain;
    std::lock_guard<std::mutex> lock(c->mu);
    if (!c->big_ready) {
        lz::HostCtx eval;
        lz::build_context(c->h.d, c->h.A, c->h.k.nu, c->h.k.split * zeta_split_scale_big(), 0, &eval);
        build_host_plan({&eval}, nullptr, &c->plain_big);
        if (c->device >= 0) {
            DeviceGuard dg(c->device);
            c->dplain_big = upload_plan(c->plain_big, &c->allocs);
        }
        c->big_ready = true;
    }
    return c->dplain_big;
}

void ensure_hess_sets(const lz_ctx* cc) {
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    if (!c->h.want_hess) throw Error{LZ_EINVAL, "context was created without Hessian tables (deriv_order < 2)"};
    std::lock_guard<std::mutex> lock(c->mu);
    lz::build_hess_sets(c->h);
}

void ensure_hess(const lz_ctx* cc) {
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    ensure_hess_sets(cc);
    std::lock_guard<std::mutex> lock(c->mu);
    if (c->hess_ready) return;
    const double sc = zeta_split_scale();
    if (sc != 1.0) {
        lz::HostCtx eval;
        lz::build_context(c->h.d, c->h.A, c->h.k.nu, c->h.k.split * sc, 2, &eval);
        lz::build_hess_sets(eval);
        build_host_plan({}, &eval, &c->hessp);
    } else {
        build_host_plan({}, &c->h, &c->hessp);
    }
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        c->dhess = upload_plan(c->hessp, &c->allocs);
    }
    c->hess_ready = true;
}

}  // namespace

int lz_ctx_create(const lz_ctx_params* p, int device, lz_ctx** out) {
    *out = nullptr;
    lz_ctx* c = new lz_ctx();
    int rc = guarded([&] {
        {
            PhaseTimer pt("ctx build_context");
            lz::build_context(p->d, p->a, p->nu, p->splitting, p->deriv_order, &c->h);
        }
        c->device = device;
        if (device >= 0) {
            int n = 0;
            if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
                cudaGetLastError();
                throw Error{LZ_ECUDA, "no such CUDA device"};
            }
        }
    });
    if (rc != LZ_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return LZ_OK;
}

int lz_ctx_prepare(const lz_ctx* c, int what) {
    return guarded([&] {
        if (what & 1) ensure_plain(c);
        if (what & 2) ensure_hess(c);
        if (what & 4) ensure_hess_sets(c);
    });
}

int lz_ctx_destroy(lz_ctx* c) {
    if (!c) return LZ_OK;
    if (c->device >= 0) {
        int old = -1;
        cudaGetDevice(&old);
        cudaSetDevice(c->device);
        free_all(&c->allocs);
        if (old >= 0) cudaSetDevice(old);
    }
    delete c;
    return LZ_OK;
}

int lz_ctx_get_info(const lz_ctx* c, lz_ctx_info* o) {
    std::memset(o, 0, sizeof(*o));
    const lz::CtxConst& k = c->h.k;
    o->d = c->h.d;
    o->branch = k.branch;
    o->log_m = k.log_m;
    o->pole = k.pole;
    o->nu = k.nu;
    o->vol = k.vol;
    o->split = k.split;
    o->s_rec = k.s;
    o->pref = k.pref;
    o->rfac = k.rfac;
    o->bconst = k.bconst;
    o->kmax = c->h.kmax;
    o->singular_coef = k.sing_coef;
    o->const_value = k.const_value;
    o->n_dir = int64_t(c->h.dir_w.size());
    o->n_rec = int64_t(c->h.rec_q.size() / c->h.d);
    o->n_dir_h = int64_t(c->h.hdir_w.size());  // 0 until the Hessian sets are built (lazy)
    o->n_rec_h = int64_t(c->h.hrec_q.size() / c->h.d);
    // table statistics are reported once the tables exist (lz_ctx_prepare)
    o->table_x_lo = c->plain.tab.x_lo;
    o->table_x_hi = c->plain.tab.x_hi;
    o->table_max_rel_err = std::max(c->plain.tab.max_rel_err, c->hessp.tab.max_rel_err);
    o->table_pieces = c->plain.tab.npieces;
    o->table_bins = c->plain.tab.nbins;
    return LZ_OK;
}

int lz_ctx_get_points(const lz_ctx* c, int which, double* dst, int64_t cap, int64_t* size) {
    if (which >= 3 && which <= 5) {
        int rc = guarded([&] { ensure_hess_sets(c); });
        if (rc != LZ_OK) return rc;
    }
    const std::vector<double>* v = nullptr;
    switch (which) {
        case 0: v = &c->h.dir_z; break;
        case 1: v = &c->h.dir_w; break;
        case 2: v = &c->h.rec_q; break;
        case 3: v = &c->h.hdir_z; break;
        case 4: v = &c->h.hdir_w; break;
        case 5: v = &c->h.hrec_q; break;
        case 6: v = &c->h.dir_n; break;
        default: return set_err(LZ_EINVAL, "unknown point set");
    }
    *size = int64_t(v->size());
    if (dst) std::memcpy(dst, v->data(), sizeof(double) * size_t(std::min<int64_t>(cap, *size)));
    return LZ_OK;
}

int lz_zeta(const lz_ctx* c, const double* k, int64_t n, double* out, uint32_t flags, int lanes, int* status,
            void* stream) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables (created with device < 0)"};
        const lz::DevPlan& P = plain_plan_for(c, n);
        DeviceGuard dg(c->device);
        int G = lanes > 0 ? lanes : auto_lanes(n);
        if (G & (G - 1) || G > 32) throw Error{LZ_EINVAL, "lanes_per_point must be a power of two <= 32"};
        check_launch(lz::launch_batch(P, false, k, n, out, flags, G, status, (cudaStream_t)stream), "zeta kernel launch", (cudaStream_t)stream);
    });
}

int lz_zeta_host(const lz_ctx* c, const double* k, int64_t n, double* out, uint32_t flags) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables (created with device < 0)"};
        for (int64_t i = 0; i < n * c->h.d; ++i)
            if (!std::isfinite(k[i])) throw Error{LZ_ENONFINITE, "k contains non-finite entries"};
        if (n == 0) return;
        const lz::DevPlan& P = plain_plan_for(c, n);
        DeviceGuard dg(c->device);
        Arena& A = arena(c->device);
        std::lock_guard<std::mutex> lock(A.mu);
        const size_t kb = sizeof(double) * size_t(n) * c->h.d, ob = sizeof(double) * size_t(n);
        A.ensure(al256(kb) + al256(ob) + 256, std::max(kb, ob) + 256);
        double* dk = reinterpret_cast<double*>(A.dbuf);
        double* dout = reinterpret_cast<double*>(A.dbuf + al256(kb));
        int* dstat = reinterpret_cast<int*>(A.dbuf + al256(kb) + al256(ob));
        check_cuda(cudaMemsetAsync(dstat, 0, sizeof(int), A.st), "memset");
        h2d(dk, k, kb, A.hbuf, A.st);
        check_launch(lz::launch_batch(P, false, dk, n, dout, flags, auto_lanes(n), dstat, A.st), "zeta kernel", A.st);
        const bool pinned_out = is_pinned(out);
        copy_d2h(pinned_out ? (void*)out : (void*)A.hbuf, dout, ob, A.st);
        int* hstat = reinterpret_cast<int*>(A.hbuf + al256(ob));
        copy_d2h(hstat, dstat, sizeof(int), A.st);
        check_cuda(cudaStreamSynchronize(A.st), "sync");
        if (!pinned_out) std::memcpy(out, A.hbuf, ob);
        if (*hstat & 1)
            throw Error{LZ_EPOLE, "Epstein zeta has a simple pole at nu = d for k in the reciprocal lattice"};
    });
}

int lz_zeta_hessian(const lz_ctx* c, const double* k, int64_t n, double* out, int lanes, void* stream) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables"};
        ensure_hess(c);
        DeviceGuard dg(c->device);
        int G = lanes > 0 ? lanes : auto_lanes(n);
        check_launch(lz::launch_batch(c->dhess, true, k, n, out, 1u, G, nullptr, (cudaStream_t)stream), "hessian kernel launch", (cudaStream_t)stream);
    });
}

int lz_zeta_hessian_host(const lz_ctx* c, const double* k, int64_t n, double* out) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables"};
        for (int64_t i = 0; i < n * c->h.d; ++i)
            if (!std::isfinite(k[i])) throw Error{LZ_ENONFINITE, "k contains non-finite entries"};
        if (n == 0) return;
        ensure_hess(c);
        DeviceGuard dg(c->device);
        const int d = c->h.d, ns = d * (d + 1) / 2;
        Arena& A = arena(c->device);
        std::lock_guard<std::mutex> lock(A.mu);
        const size_t kb = sizeof(double) * size_t(n) * d, ob = sizeof(double) * size_t(n) * ns;
        A.ensure(al256(kb) + al256(ob), std::max(kb, ob) + 256);
        double* dk = reinterpret_cast<double*>(A.dbuf);
        double* dout = reinterpret_cast<double*>(A.dbuf + al256(kb));
        h2d(dk, k, kb, A.hbuf, A.st);
        check_launch(lz::launch_batch(c->dhess, true, dk, n, dout, 1u, auto_lanes(n), nullptr, A.st), "hessian kernel", A.st);
        copy_d2h(A.hbuf, dout, ob, A.st);
        check_cuda(cudaStreamSynchronize(A.st), "sync");
        std::memcpy(out, A.hbuf, ob);
    });
}

}  // extern "C"

namespace {

// Multi-indices |alpha| = order in the reference's order (L/epstein.py:426-433, head ascending);
// the kernel's compile-time list (deriv.cu DerivSpec) enumerates the same way.
std::vector<int> multi_indices(int d, int order) {
    std::vector<int> out;
    int total = 1;
    for (int a = 0; a < d; ++a) total *= order + 1;
    std::vector<int> cur(d);
    for (int c = 0; c < total; ++c) {
        int rem = c, sum = 0;
        for (int a = d - 1; a >= 0; --a) {
            cur[a] = rem % (order + 1);
            rem /= order + 1;
            sum += cur[a];
        }
        if (sum == order) out.insert(out.end(), cur.begin(), cur.end());
    }
    return out;
}

// Order-m derivative plan of a context: direct weights 2 (2 pi)^m w z^alpha, reciprocal points
// sorted by |q|, tables of F^{(j)} = (-1)^j c^{s+j} E_{1-s-j}, j = ceil(m/2) .. m.
const lz::DevDeriv& ensure_deriv(const lz_ctx* cc, int order) {
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    std::lock_guard<std::mutex> lock(c->mu);
    auto it = c->dderiv.find(order);
    if (it != c->dderiv.end()) return it->second;
    const lz::HostCtx& h = c->h;
    const int d = h.d;
    if (h.k.branch == lz::kTrivial) throw Error{LZ_EINVAL, "derivatives of a trivial-branch zeta are zero"};
    std::vector<double> dir_n, rec_n;
    lz::build_deriv_sets(h, order, &dir_n, &rec_n);
    const std::vector<int> alphas = multi_indices(d, order);
    const int na = int(alphas.size()) / d;
    const size_t nd = dir_n.size() / d;
    std::vector<double> W(nd * na);
    const ld twopi_m = std::pow(2.0L * ld(lz::kPi), ld(order));
    for (size_t i = 0; i < nd; ++i) {
        ld z[lz::kMaxDim];
        const ld w = direct_weight(h, &dir_n[i * d], z);
        for (int j = 0; j < na; ++j) {
            ld v = 2.0L * twopi_m * w;
            for (int a = 0; a < d; ++a)
                for (int e = 0; e < alphas[j * d + a]; ++e) v *= z[a];
            W[i * na + j] = double(v);
        }
    }
    const size_t nr = rec_n.size() / d;
    std::vector<double> q(nr * d);
    std::vector<ld> qn(nr);
    for (size_t i = 0; i < nr; ++i) {
        ld r2 = 0.0L;
        for (int a = 0; a < d; ++a) {
            ld v = 0.0L;
            for (int b = 0; b < d; ++b) v += ld(h.B[a * d + b]) * rec_n[i * d + b];
            q[i * d + a] = double(v);
            r2 += v * v;
        }
        qn[i] = std::sqrt(r2);
    }
    std::vector<size_t> ord(nr);
    for (size_t i = 0; i < nr; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return qn[a] < qn[b]; });
    std::vector<double> rq(nr * d), rn(nr);
    for (size_t i = 0; i < nr; ++i) {
        for (int a = 0; a < d; ++a) rq[i * d + a] = q[ord[i] * d + a];
        rn[i] = double(qn[ord[i]]);
    }
    const int j0 = (order + 1) / 2, nf = lz::deriv_nfunc(order);
    double p[4], sc[4];
    const ld cl = ld(lz::kPi) / ld(h.k.split);
    for (int j = 0; j < nf; ++j) {
        const int jj = j0 + j;
        p[j] = 1.0 - h.k.s - jj;
        sc[j] = double(((jj & 1) ? -1.0L : 1.0L) * std::pow(cl, ld(h.k.s) + jj));
    }
    lz::HostTable& tab = c->dtab[order];
    const double rp = std::fabs(h.k.rfac * h.k.pref);
    if (nr > 0) lz::build_table(p, sc, nf, double(cl), lz::table_x_lo(h), rp, &tab, std::max(1.0, order / 2.0));
    else tab.nfunc = nf;
    lz::DevDeriv P;
    std::memset(&P, 0, sizeof(P));
    P.d = d;
    P.order = order;
    P.n_dir = int(nd);
    P.n_rec = int(nr);
    std::memcpy(P.A, h.A, sizeof(P.A));
    std::memcpy(P.B, h.B, sizeof(P.B));
    P.pref = h.k.pref;
    P.rfac = h.k.rfac;
    P.r_cut = nr > 0 ? double(std::sqrt(ld(tab.x_hi) / cl) * (1.0L + 1e-9L)) : 0.0;
    {
        DeviceGuard dg(c->device);
        P.dir_n = upload(dir_n, &c->allocs);
        P.dir_w = upload(W, &c->allocs);
        P.rec_q = upload(rq, &c->allocs);
        P.rec_norm = upload(rn, &c->allocs);
        P.tab.dir = upload(tab.dir, &c->allocs);
        P.tab.coef = upload(tab.coef, &c->allocs);
    }
    P.tab.nbins = tab.nbins;
    P.tab.nfunc = nf;
    P.tab.npieces = tab.npieces;
    P.tab.ncoef = int(tab.coef.size());
    P.tab.x_lo = tab.x_lo;
    P.tab.inv_hb = tab.inv_hb;
    P.tab.x_hi = tab.x_hi;
    P.tab.c = double(cl);
    P.tab.r_scale = double(cl) * tab.inv_hb;
    P.tab.x_off = tab.x_lo * tab.inv_hb;
    P.tab.nbins_d = double(tab.nbins);
    for (int j = 0; j < nf; ++j) {
        P.tab.p[j] = p[j];
        P.tab.scale[j] = sc[j];
    }
    return c->dderiv.emplace(order, P).first->second;
}


// Moment-form plan (deriv.cu deriv_moment_kernel) of order m (0..12, d <= 4).  taylor = 0: d^alpha Z
// at arbitrary k over the order-m point sets; taylor = 1: d^alpha Z_reg at k = 0 over the point
// sets of order set_order (L/epstein.py:376-377, the table of reg_derivatives(set_order)), the
// q = 0 term from the rho-series of t0_reg (L/epstein.py:403-413) and bconst (m = 0) in `add`.
const lz::DevDeriv& ensure_deriv_g(const lz_ctx* cc, int order, int taylor, int set_order) {
    lz_ctx* c = const_cast<lz_ctx*>(cc);
    std::lock_guard<std::mutex> lock(c->mu);
    const auto key = std::make_tuple(order, taylor, set_order);
    auto it = c->dderiv_g.find(key);
    if (it != c->dderiv_g.end()) return it->second;
    const lz::HostCtx& h = c->h;
    const int d = h.d, m = order;
    if (h.k.branch == lz::kTrivial) throw Error{LZ_EINVAL, "derivatives of a trivial-branch zeta are zero"};
    std::vector<double> dir_n, rec_n;
    lz::build_deriv_sets(h, set_order, &dir_n, &rec_n);
    const std::vector<int> alphas = multi_indices(d, m);
    const int na = int(alphas.size()) / d;
    const int j0 = (m + 1) / 2, nf = m - j0 + 1;
    if (nf > lz::kMaxFunc - 1) throw Error{LZ_EINVAL, "derivative order too high"};
    const int rs = nf + d * (m + 1);
    if (rs > 255) throw Error{LZ_EINVAL, "derivative record too large"};
    // direct set: Cartesian z and 2 (2 pi)^m w_z (long double, rounded once)
    const size_t nd = dir_n.size() / d;
    std::vector<double> dz(nd * d), dw0(nd);
    const ld twopi_m = std::pow(2.0L * ld(lz::kPi), ld(m));
    for (size_t i = 0; i < nd; ++i) {
        ld z[lz::kMaxDim];
        const ld w = direct_weight(h, &dir_n[i * d], z);
        for (int a = 0; a < d; ++a) dz[i * d + a] = double(z[a]);
        dw0[i] = double(2.0L * twopi_m * w);
    }
    // reciprocal set sorted by |q|
    const size_t nr = rec_n.size() / d;
    std::vector<double> q(nr * d);
    std::vector<ld> qn(nr);
    for (size_t i = 0; i < nr; ++i) {
        ld r2 = 0.0L;
        for (int a = 0; a < d; ++a) {
            ld v = 0.0L;
            for (int b = 0; b < d; ++b) v += ld(h.B[a * d + b]) * rec_n[i * d + b];
            q[i * d + a] = double(v);
            r2 += v * v;
        }
        qn[i] = std::sqrt(r2);
    }
    std::vector<size_t> ord(nr);
    for (size_t i = 0; i < nr; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return qn[a] < qn[b]; });
    std::vector<double> rq(nr * d), rn(nr);
    for (size_t i = 0; i < nr; ++i) {
        for (int a = 0; a < d; ++a) rq[i * d + a] = q[ord[i] * d + a];
        rn[i] = double(qn[ord[i]]);
    }
    // tables of F^{(p)} = (-1)^p c^{s+p} E_{1-s-p}, p = j0 .. m
    double p[lz::kMaxFunc] = {}, sc[lz::kMaxFunc] = {};
    const ld cl = ld(lz::kPi) / ld(h.k.split);
    for (int j = 0; j < nf; ++j) {
        const int jj = j0 + j;
        p[j] = 1.0 - h.k.s - jj;
        sc[j] = double(((jj & 1) ? -1.0L : 1.0L) * std::pow(cl, ld(h.k.s) + jj));
    }
    lz::HostTable& tab = c->dtab_g[key];
    const double rp = std::fabs(h.k.rfac * h.k.pref);
    if (nr > 0) lz::build_table(p, sc, nf, double(cl), lz::table_x_lo(h), rp, &tab, std::max(1.0, m / 2.0));
    else tab.nfunc = nf;
    // moments: one direct moment per alpha, then R[p][e], |e| = 2p - m
    auto code = [&](int fslot, const int* e) {
        unsigned long long v = (unsigned long long)fslot;
        for (int a = 0; a < d; ++a) v |= (unsigned long long)(nf + a * (m + 1) + e[a]) << (8 * (a + 1));
        return v;
    };
    std::vector<unsigned long long> mom;
    for (int ia = 0; ia < na; ++ia) mom.push_back(code(0, &alphas[ia * d]));
    std::map<std::vector<int>, int> rmap;  // (p, e) -> reciprocal moment index
    int n_rmom = 0;
    for (int pp = j0; pp <= m; ++pp) {
        const std::vector<int> es = multi_indices(d, 2 * pp - m);
        for (size_t i = 0; i < es.size() / d; ++i) {
            std::vector<int> key2 = {pp};
            key2.insert(key2.end(), es.begin() + i * d, es.begin() + (i + 1) * d);
            rmap[key2] = n_rmom++;
            mom.push_back(code(pp - j0, &es[i * d]));
        }
    }
    auto fact = [](int n) {
        double f = 1.0;
        for (int i = 2; i <= n; ++i) f *= i;
        return f;
    };
    std::vector<int> hoff(na + 1, 0), hmom;
    std::vector<double> hcoef, add;
    for (int ia = 0; ia < na; ++ia) {
        const int* al = &alphas[ia * d];
        int jv[lz::kMaxDim] = {0, 0, 0, 0};
        for (;;) {
            int js = 0;
            double cf = 1.0;
            std::vector<int> key2(1);
            for (int a = 0; a < d; ++a) {
                js += jv[a];
                cf *= fact(al[a]) / (fact(jv[a]) * fact(al[a] - 2 * jv[a]));
                key2.push_back(al[a] - 2 * jv[a]);
            }
            key2[0] = m - js;
            hmom.push_back(rmap.at(key2));
            hcoef.push_back(cf);
            int a = 0;
            while (a < d) {
                if (++jv[a] <= al[a] / 2) break;
                jv[a] = 0;
                ++a;
            }
            if (a == d) break;
        }
        hoff[ia + 1] = int(hmom.size());
    }
    if (taylor) {
        add.assign(na, 0.0);
        for (int ia = 0; ia < na; ++ia) {
            const int* al = &alphas[ia * d];
            ld v = (m == 0) ? ld(h.k.bconst) : 0.0L;
            bool even = true;
            for (int a = 0; a < d; ++a) even = even && (al[a] % 2 == 0);
            if (even) {
                const int nn = m / 2;
                ld mult = ld(fact(nn)), fac = 1.0L;
                for (int a = 0; a < d; ++a) {
                    mult /= ld(fact(al[a] / 2));
                    fac *= ld(fact(al[a]));
                }
                v += ld(h.k.rfac) * lz::t0_coeff(h.k, nn) * mult * fac;
            }
            add[ia] = double(v);
        }
    }
    lz::DevDeriv P;
    std::memset(&P, 0, sizeof(P));
    P.d = d;
    P.order = m;
    P.n_dir = int(nd);
    P.n_rec = int(nr);
    std::memcpy(P.A, h.A, sizeof(P.A));
    std::memcpy(P.B, h.B, sizeof(P.B));
    P.pref = h.k.pref;
    P.rfac = h.k.rfac;
    P.r_cut = nr > 0 ? double(std::sqrt(ld(tab.x_hi) / cl) * (1.0L + 1e-9L)) : 0.0;
    P.n_alpha = na;
    P.n_dmom = na;
    P.n_rmom = n_rmom;
    P.nf = nf;
    P.rs = rs;
    P.taylor = taylor;
    {
        DeviceGuard dg(c->device);
        P.dir_n = upload(dir_n, &c->allocs);
        P.dir_z = upload(dz, &c->allocs);
        P.dir_w0 = upload(dw0, &c->allocs);
        P.rec_q = upload(rq, &c->allocs);
        P.rec_norm = upload(rn, &c->allocs);
        P.tab.dir = upload(tab.dir, &c->allocs);
        P.tab.coef = upload(tab.coef, &c->allocs);
        P.mom = upload(mom, &c->allocs);
        P.hoff = upload(hoff, &c->allocs);
        P.hmom = upload(hmom, &c->allocs);
        P.hcoef = upload(hcoef, &c->allocs);
        if (taylor) P.add = upload(add, &c->allocs);
    }
    P.tab.nbins = tab.nbins;
    P.tab.nfunc = nf;
    P.tab.npieces = tab.npieces;
    P.tab.ncoef = int(tab.coef.size());
    P.tab.x_lo = tab.x_lo;
    P.tab.inv_hb = tab.inv_hb;
    P.tab.x_hi = tab.x_hi;
    P.tab.c = double(cl);
    P.tab.r_scale = double(cl) * tab.inv_hb;
    P.tab.x_off = tab.x_lo * tab.inv_hb;
    P.tab.nbins_d = double(tab.nbins);
    for (int j = 0; j < nf; ++j) {
        P.tab.p[j] = p[j];
        P.tab.scale[j] = sc[j];
    }
    return c->dderiv_g.emplace(key, P).first->second;
}

// compile-time kernel (orders 1..4, d <= 3) unless LATSUM_DERIV_MOMENTS=1; the moment form otherwise
bool deriv_use_fixed(int d, int order) {
    static const int force = [] {
        const char* e = std::getenv("LATSUM_DERIV_MOMENTS");
        return e ? std::atoi(e) : 0;
    }();
    return !force && order >= 1 && order <= 4 && d <= 3;
}

cudaError_t launch_derivatives(const lz_ctx* c, int order, const double* k, int64_t n, double* out, int* status,
                               cudaStream_t st) {
    if (deriv_use_fixed(c->h.d, order)) return lz::launch_deriv(ensure_deriv(c, order), k, n, out, status, st);
    return lz::launch_deriv_g(ensure_deriv_g(c, order, 0, order), k, n, out, status, st);
}
}  // namespace

extern "C" {

int lz_multi_indices(int d, int order, int* alphas, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (d < 1 || d > 4 || order < 0) throw Error{LZ_EINVAL, "bad dimension or order"};
        const std::vector<int> a = multi_indices(d, order);
        *n = int64_t(a.size()) / d;
        for (int64_t i = 0; i < std::min<int64_t>(cap, *n) * d; ++i) alphas[i] = a[size_t(i)];
    });
}

int lz_zeta_derivatives(const lz_ctx* c, int order, const double* k, int64_t n, double* out, int* status,
                        void* stream) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables"};
        if (order < 1 || order > 12) throw Error{LZ_EINVAL, "derivative order must be 1..12"};
        DeviceGuard dg(c->device);
        check_launch(launch_derivatives(c, order, k, n, out, status, (cudaStream_t)stream), "derivative kernel", (cudaStream_t)stream);
    });
}

int lz_zeta_derivatives_host(const lz_ctx* c, int order, const double* k, int64_t n, double* out) {
    return guarded([&] {
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables"};
        if (order < 1 || order > 12) throw Error{LZ_EINVAL, "derivative order must be 1..12"};
        for (int64_t i = 0; i < n * c->h.d; ++i)
            if (!std::isfinite(k[i])) throw Error{LZ_ENONFINITE, "k contains non-finite entries"};
        if (n == 0) return;
        DeviceGuard dg(c->device);
        const int d = c->h.d, na = lz::deriv_count(d, order);
        Arena& A = arena(c->device);
        std::lock_guard<std::mutex> lock(A.mu);
        const size_t kb = sizeof(double) * size_t(n) * d, ob = sizeof(double) * size_t(n) * na;
        A.ensure(al256(kb) + al256(ob) + 256, std::max(kb, ob) + 256);
        double* dk = reinterpret_cast<double*>(A.dbuf);
        double* dout = reinterpret_cast<double*>(A.dbuf + al256(kb));
        int* dstat = reinterpret_cast<int*>(A.dbuf + al256(kb) + al256(ob));
        check_cuda(cudaMemsetAsync(dstat, 0, sizeof(int), A.st), "memset");
        h2d(dk, k, kb, A.hbuf, A.st);
        check_launch(launch_derivatives(c, order, dk, n, dout, dstat, A.st), "derivative kernel", A.st);
        copy_d2h(A.hbuf, dout, ob, A.st);
        int* hstat = reinterpret_cast<int*>(A.hbuf + al256(ob));
        copy_d2h(hstat, dstat, sizeof(int), A.st);
        check_cuda(cudaStreamSynchronize(A.st), "sync");
        std::memcpy(out, A.hbuf, ob);
        if (*hstat & 1) throw Error{LZ_EPOLE, "derivatives of Z are singular at k in the reciprocal lattice"};
    });
}

int lz_grid_tiles(int d, const lz_grid* g, int64_t* n_nodes, int64_t* n_tiles) {
    return guarded([&] {
        if (d < 1 || d > 4) throw Error{LZ_EINVAL, "dimension outside 1..4"};
        lz::DevGrid dg;
        lz_grid all = *g;
        all.tile_lo = 0;
        all.tile_hi = 0;
        fill_grid(d, &all, &dg);
        *n_nodes = int64_t(dg.n_cell) * dg.n_u * (d > 1 ? dg.n_v : 1) * (d > 2 ? dg.n_v : 1);
        *n_tiles = dg.tile_hi;
    });
}

int lz_plan_create_product(const lz_ctx* const* ctxs, const int* mult, int nctx, lz_plan** out) {
    *out = nullptr;
    lz_plan* pl = new lz_plan();
    int rc = guarded([&] {
        if (nctx < 1 || nctx > lz::kMaxCtx) throw Error{LZ_EINVAL, "product plans fuse 1..4 distinct exponents"};
        std::vector<const lz::HostCtx*> plain;
        for (int j = 0; j < nctx; ++j) {
            if (ctxs[j]->h.k.branch == lz::kTrivial)
                throw Error{LZ_EINVAL, "trivial-branch factors are constants; fold them on the host"};
            if (mult[j] < 1) throw Error{LZ_EINVAL, "multiplicities must be >= 1"};
            plain.push_back(&ctxs[j]->h);
            pl->mult[j] = mult[j];
        }
        pl->device = ctxs[0]->device;  // < 0: host tables only (inspection / tests)
        pl->d = ctxs[0]->h.d;
        if (pl->d > 3) throw Error{LZ_EINVAL, "integral kernels support d <= 3"};
        pl->kind = 0;
        build_host_plan(plain, nullptr, &pl->hp);
        if (pl->device >= 0) {
            DeviceGuard dg(pl->device);
            pl->P = upload_plan(pl->hp, &pl->allocs);
        }
    });
    if (rc != LZ_OK) {
        free_all(&pl->allocs);
        delete pl;
        return rc;
    }
    *out = pl;
    return LZ_OK;
}

int lz_plan_create_atm(const lz_ctx* z3, const lz_ctx* z5, lz_plan** out) {
    *out = nullptr;
    lz_plan* pl = new lz_plan();
    int rc = guarded([&] {
        if (!z5->h.want_hess) throw Error{LZ_EINVAL, "the nu = 5 context needs deriv_order >= 2"};
        ensure_hess_sets(z5);
        if (z3->h.k.branch == lz::kTrivial || z5->h.k.branch == lz::kTrivial)
            throw Error{LZ_EINVAL, "ATM contexts cannot be trivial"};
        pl->device = z3->device;  // < 0: host tables only (inspection / tests)
        pl->d = z3->h.d;
        if (pl->d > 3) throw Error{LZ_EINVAL, "ATM is defined for d <= 3"};
        pl->kind = 1;
        if (std::fabs(z5->h.k.nu - z3->h.k.nu - 2.0) > 1e-12)
            throw Error{LZ_EINVAL, "ATM plan needs exponents nu and nu + 2 (Z_3 and the Hessian of Z_5)"};
        {
            PhaseTimer pt("atm build_host_plan");
            build_host_plan({&z3->h}, &z5->h, &pl->hp, /*trace_z=*/true);
        }
        if (!pl->hp.alias_fp) throw Error{LZ_EINVAL, "ATM plan: F' alias expected"};
        if (pl->device >= 0) {
            PhaseTimer pt("atm upload_plan");
            DeviceGuard dg(pl->device);
            pl->P = upload_plan(pl->hp, &pl->allocs);
        }
    });
    if (rc != LZ_OK) {
        free_all(&pl->allocs);
        delete pl;
        return rc;
    }
    *out = pl;
    return LZ_OK;
}

int lz_plan_destroy(lz_plan* pl) {
    if (!pl) return LZ_OK;
    if (pl->device >= 0) {
        int old = -1;
        cudaGetDevice(&old);
        cudaSetDevice(pl->device);
        free_all(&pl->allocs);
        if (old >= 0) cudaSetDevice(old);
    }
    delete pl;
    return LZ_OK;
}

int lz_plan_integrate(const lz_plan* pl, const lz_grid* g, double* partials, int grid_blocks, void* stream) {
    return guarded([&] {
        if (pl->device < 0) throw Error{LZ_ECUDA, "plan has no device tables (created from host-only contexts)"};
        DeviceGuard dg(pl->device);
        lz::DevGrid dgd;
        fill_grid(pl->d, g, &dgd);
        PhaseTimer pt_ga("integrate grid+scratch");
        const GridArrays& ga = grid_arrays(pl, g);
        dgd.u = ga.u;
        dgd.wu = ga.wu;
        dgd.v = ga.v;
        dgd.wv = ga.wv;
        cudaStream_t st = (cudaStream_t)stream;
        {
            lz_grid full = *g;
            full.tile_lo = full.tile_hi = 0;
            lz::DevGrid tmp;
            fill_grid(pl->d, &full, &tmp);
            const bool need_wpart = pl->kind != 1 || lz::atm_needs_wpart(pl->P, dgd);
            // row-factorised ATM plans: the D table of this grid's radial nodes (kernels.cu row_table_kernel)
            const size_t dbytes = pl->kind == 1 && pl->P.row_on
                                      ? size_t(3) * size_t(dgd.n_u) * size_t(pl->P.row_nJ) * size_t(pl->P.row_NI) * 16
                                      : 0;
            dgd.dtab = nullptr;
            tile_scratch(pl->device, st, (tmp.n_patch + 7) / 8, need_wpart, &dgd.wpart, &dgd.tcount, &dgd.work,
                         dbytes, &dgd.dtab);
        }
        if (pl->kind == 0)
            check_launch(lz::launch_product(pl->P, dgd, pl->mult, partials, grid_blocks, st), "product kernel", st);
        else
            check_launch(lz::launch_atm(pl->P, dgd, partials, grid_blocks, st), "atm kernel", st);
    });
}

int lz_plan_product_at(const lz_plan* pl, const double* k, int64_t n, double* out, int* status, void* stream) {
    return guarded([&] {
        if (pl->kind != 0) throw Error{LZ_EINVAL, "lz_plan_product_at needs a product plan"};
        DeviceGuard dg(pl->device);
        const int4 m = make_int4(pl->mult[0], pl->mult[1], pl->mult[2], pl->mult[3]);
        check_launch(lz::launch_product_at(pl->P, m, k, n, out, auto_lanes(n), status, (cudaStream_t)stream), "product kernel", (cudaStream_t)stream);
    });
}

int lz_plan_get_info(const lz_plan* pl, lz_plan_info* o) {
    std::memset(o, 0, sizeof(*o));
    o->d = pl->d;
    o->kind = pl->kind;
    o->nctx = pl->hp.nctx;
    o->hess = pl->hp.hess;
    o->alias = pl->hp.alias_fp;
    o->n_dir = int64_t(pl->hp.dir_n.size() / std::max(pl->d, 1));
    o->n_runs = int64_t(pl->hp.run_info.size() / 2);
    o->n_rec = int64_t(pl->hp.rec_norm.size());
    o->n_funcs = pl->hp.tab.nfunc;
    o->table_pieces = pl->hp.tab.npieces;
    o->table_bins = pl->hp.tab.nbins;
    o->table_x_lo = pl->hp.tab.x_lo;
    o->table_x_hi = pl->hp.tab.x_hi;
    o->table_max_rel_err = pl->hp.tab.max_rel_err;
    o->r_cut = pl->hp.r_cut;
    o->split = pl->hp.c > 0 ? lz::kPi / pl->hp.c : 0.0;
    o->n_t0 = pl->hp.n_t0;
    o->t0_rho_max = pl->hp.t0_rho_max;
    const size_t ns = pl->hp.nctx + (pl->hp.hess ? 2 : 0);
    o->smem_bytes = int64_t(8 * (pl->hp.direct.size() + pl->hp.rec_q.size() +
                                 pl->hp.rec_norm.size() + pl->hp.tab.coef.size() + ns * lz::kT0) +
                            4 * pl->hp.tab.dir.size());
    return LZ_OK;
}

// Device that owns a device pointer (multi-GPU processes: the library's own current device
// may differ from the caller's).
static int device_of(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return at.type == cudaMemoryTypeDevice ? at.device : -1;
}

int lz_reduce_partials(const double* partials, int64_t n_tiles, int ncomp, double* out, void* stream) {
    return guarded([&] {
        DeviceGuard dg(device_of(partials));
        check_launch(lz::launch_reduce(partials, n_tiles, ncomp, out, (cudaStream_t)stream), "reduce kernel", (cudaStream_t)stream);
    });
}

int lz_reduce_chunks(const double* partials, int64_t n_tiles, int ncomp, int64_t chunk_tiles, int64_t chunk_lo,
                     int64_t chunk_hi, double* chunk_out, void* stream) {
    return guarded([&] {
        if (n_tiles < 0 || ncomp < 1 || chunk_tiles < 1 || chunk_lo < 0 || chunk_hi < chunk_lo ||
            chunk_hi * chunk_tiles >= n_tiles + chunk_tiles)
            throw Error{LZ_EINVAL, "chunk range outside the tile vector"};
        if (chunk_hi == chunk_lo) return;
        DeviceGuard dg(device_of(partials));
        check_launch(lz::launch_chunks(partials, n_tiles, ncomp, chunk_tiles, chunk_lo, chunk_hi, chunk_out,
                                     (cudaStream_t)stream), "chunk kernel", (cudaStream_t)stream);
    });
}

int lz_chunk_layout(int64_t n_tiles, int64_t* chunk_tiles, int64_t* n_chunks) {
    constexpr int64_t kMaxChunks = 96;
    const int64_t ct = std::max<int64_t>(1, (n_tiles + kMaxChunks - 1) / kMaxChunks);
    if (chunk_tiles) *chunk_tiles = ct;
    if (n_chunks) *n_chunks = n_tiles > 0 ? (n_tiles + ct - 1) / ct : 0;
    return LZ_OK;
}

int lz_transfer_stats(int64_t* h2d_bytes, int64_t* d2h_bytes, int reset) {
    if (h2d_bytes) *h2d_bytes = g_h2d_bytes.load();
    if (d2h_bytes) *d2h_bytes = g_d2h_bytes.load();
    if (reset) {
        g_h2d_bytes = 0;
        g_d2h_bytes = 0;
    }
    return LZ_OK;
}

int lz_release_caches(int device) {
    return guarded([&] {
        int old = -1;
        check_cuda(cudaGetDevice(&old), "cudaGetDevice");
        auto on = [&](int dev) { return device < 0 || dev == device; };
        {
            std::lock_guard<std::mutex> lock(g_grid_mu);
            for (auto it = g_grid_cache.begin(); it != g_grid_cache.end();) {
                if (on(std::get<0>(it->first))) {
                    cudaSetDevice(std::get<0>(it->first));
                    cudaDeviceSynchronize();
                    cudaFree(const_cast<double*>(it->second.u));  // one allocation per entry
                    it = g_grid_cache.erase(it);
                } else {
                    ++it;
                }
            }
        }
        {
            std::lock_guard<std::mutex> lock(g_scratch_mu);
            for (auto it = g_scratch.begin(); it != g_scratch.end();) {
                if (on(it->first.first)) {
                    cudaSetDevice(it->first.first);
                    cudaDeviceSynchronize();
                    if (it->second.wpart) cudaFree(it->second.wpart);
                    if (it->second.dtab) cudaFree(it->second.dtab);
                    if (it->second.tcount) cudaFree(it->second.tcount);
                    it = g_scratch.erase(it);
                } else {
                    ++it;
                }
            }
        }
        {
            std::lock_guard<std::mutex> lock(g_arena_mu);
            for (auto& kv : g_arenas) {
                if (!on(kv.first) || !kv.second) continue;
                Arena& a = *kv.second;
                std::lock_guard<std::mutex> al(a.mu);
                cudaSetDevice(kv.first);
                cudaDeviceSynchronize();
                if (a.dbuf) cudaFree(a.dbuf);
                if (a.hbuf) cudaFreeHost(a.hbuf);
                a.dbuf = a.hbuf = nullptr;
                a.dcap = a.hcap = 0;
            }
        }
        if (old >= 0) cudaSetDevice(old);
        check_cuda(cudaGetLastError(), "release caches");
    });
}

int lz_plan_integrate_host(const lz_plan* pl, const lz_grid* g, double* out) {
    return guarded([&] {
        if (pl->device < 0) throw Error{LZ_ECUDA, "plan has no device tables (created from host-only contexts)"};
        DeviceGuard dg(pl->device);
        int64_t n_nodes = 0, n_tiles = 0;
        int rc = lz_grid_tiles(pl->d, g, &n_nodes, &n_tiles);
        if (rc != LZ_OK) throw Error{rc, g_last_error};
        const int ncomp = pl->kind == 0 ? 1 : 2;
        // the same reduction as the sharded path (tiles -> fixed chunks -> total), so one-call and
        // multi-rank results carry the same bits
        int64_t chunk_tiles = 0, n_chunks = 0;
        lz_chunk_layout(n_tiles, &chunk_tiles, &n_chunks);
        Arena& A = arena(pl->device);
        std::lock_guard<std::mutex> lock(A.mu);
        const size_t pb = sizeof(double) * size_t(n_tiles) * ncomp;
        const size_t cb = sizeof(double) * size_t(n_chunks) * ncomp;
        A.ensure(al256(pb) + al256(cb) + 256, 256);
        double* dp = reinterpret_cast<double*>(A.dbuf);
        double* dc = reinterpret_cast<double*>(A.dbuf + al256(pb));
        double* dout = reinterpret_cast<double*>(A.dbuf + al256(pb) + al256(cb));
        lz_grid gg = *g;
        gg.tile_lo = 0;
        gg.tile_hi = 0;
        rc = lz_plan_integrate(pl, &gg, dp, 0, A.st);
        if (rc != LZ_OK) throw Error{rc, g_last_error};
        check_launch(lz::launch_chunks(dp, n_tiles, ncomp, chunk_tiles, 0, n_chunks, dc, A.st), "chunk reduce", A.st);
        check_launch(lz::launch_reduce(dc, n_chunks, ncomp, dout, A.st), "reduce", A.st);
        copy_d2h(A.hbuf, dout, sizeof(double) * ncomp, A.st);
        check_cuda(cudaStreamSynchronize(A.st), "sync");
        std::memcpy(out, A.hbuf, sizeof(double) * ncomp);
    });
}

int lz_ctx_reg_derivatives(const lz_ctx* c, int order, int* alphas, double* vals, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (order < 0 || order % 2 || order > 12) throw Error{LZ_EINVAL, "derivative order must be even and <= 12"};
        std::vector<int> al;
        std::vector<double> v;
        lz::build_reg_derivatives(c->h, order, &al, &v);
        *n = int64_t(v.size());
        const int64_t m = std::min<int64_t>(cap, *n);
        if (alphas && m > 0) std::memcpy(alphas, al.data(), sizeof(int) * size_t(m) * c->h.d);
        if (vals && m > 0) std::memcpy(vals, v.data(), sizeof(double) * size_t(m));
    });
}

// Device Taylor tables (deriv.cu moment kernel in Taylor mode): every even total order <= order,
// one single-point launch per order over the order-`order` point sets (L/epstein.py:376-377).
int lz_ctx_reg_derivatives_device(const lz_ctx* c, int order, int* alphas, double* vals, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (order < 0 || order % 2 || order > 12) throw Error{LZ_EINVAL, "derivative order must be even and <= 12"};
        if (c->device < 0) throw Error{LZ_ECUDA, "context has no device tables"};
        const int d = c->h.d;
        std::vector<int> al;
        for (int total = 0; total <= order; total += 2) {
            const std::vector<int> a = multi_indices(d, total);
            al.insert(al.end(), a.begin(), a.end());
        }
        const int64_t na = int64_t(al.size()) / d;
        std::vector<double> v(size_t(na), 0.0);
        if (c->h.k.branch == lz::kTrivial) {
            v[0] = c->h.k.const_value;  // total order 0 comes first
        } else {
            DeviceGuard dg(c->device);
            Arena& A = arena(c->device);
            std::lock_guard<std::mutex> lock(A.mu);
            const size_t ob = sizeof(double) * size_t(na);
            A.ensure(al256(ob) + 256, ob + 256);
            double* dout = reinterpret_cast<double*>(A.dbuf);
            int64_t off = 0;
            for (int total = 0; total <= order; total += 2) {
                const lz::DevDeriv& P = ensure_deriv_g(c, total, 1, order);
                check_launch(lz::launch_deriv_g(P, nullptr, 1, dout + off, nullptr, A.st), "taylor kernel", A.st);
                off += P.n_alpha;
            }
            copy_d2h(A.hbuf, dout, ob, A.st);
            check_cuda(cudaStreamSynchronize(A.st), "sync");
            std::memcpy(v.data(), A.hbuf, ob);
        }
        *n = na;
        const int64_t m = std::min<int64_t>(cap, na);
        if (alphas && m > 0) std::memcpy(alphas, al.data(), sizeof(int) * size_t(m) * d);
        if (vals && m > 0) std::memcpy(vals, v.data(), sizeof(double) * size_t(m));
    });
}

double lz_upper_gamma(double s, double x) {
    if (!(x > 0.0)) return std::nan("");
    return double(lz::upper_gamma<long double>(s, x));
}

int lz_direct_sum3(int device, int d, const double* a, int64_t L, int kind, const double* nus, double max_pairs,
                   double* out) {
    return guarded([&] {
        if (d < 1 || d > 3) throw Error{LZ_EINVAL, "direct sums support d = 1..3"};
        if (L < 1) throw Error{LZ_EINVAL, "truncation L must be >= 1"};
        if (kind != 0 && kind != 1) throw Error{LZ_EINVAL, "kind: 0 three-body zeta, 1 ATM energy"};
        int64_t npts = 1;
        for (int i = 0; i < d; ++i) npts *= 2 * L + 1;
        const double pairs = double(npts) * double(npts);
        if (max_pairs > 0 && pairs > max_pairs)
            throw Error{LZ_EINVAL, "direct sum exceeds the term guard (pass a larger max_pairs)"};
        DeviceGuard guard(device);
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "device");
        Arena& ar = arena(dev);
        std::lock_guard<std::mutex> lock(ar.mu);
        const int64_t nblocks = (npts + lz::direct_tile() - 1) / lz::direct_tile();
        ar.ensure(al256(sizeof(double) * 16) + al256(sizeof(double) * size_t(nblocks)) + 256, 256);
        double* dA = reinterpret_cast<double*>(ar.dbuf);
        double* dp = reinterpret_cast<double*>(ar.dbuf + al256(sizeof(double) * 16));
        double* dout = reinterpret_cast<double*>(ar.dbuf + al256(sizeof(double) * 16) +
                                                 al256(sizeof(double) * size_t(nblocks)));
        double hA[16] = {0};
        for (int i = 0; i < d * d; ++i) hA[i] = a[i];
        copy_h2d(dA, hA, sizeof(hA), ar.st);
        const double nz[3] = {nus ? nus[0] : 0.0, nus ? nus[1] : 0.0, nus ? nus[2] : 0.0};
        check_launch(lz::launch_direct(d, kind, L, npts, dA, nz, dp, nblocks, ar.st), "direct kernel", ar.st);
        check_launch(lz::launch_reduce(dp, nblocks, 1, dout, ar.st), "reduce", ar.st);
        copy_d2h(ar.hbuf, dout, sizeof(double), ar.st);
        check_cuda(cudaStreamSynchronize(ar.st), "sync");
        double v;
        std::memcpy(&v, ar.hbuf, sizeof(double));
        *out = kind == 1 ? v / 6.0 : v;
    });
}

int lz_allreduce_partials(double* partials, int64_t n, void* nccl_comm, void* stream) {
    return guarded([&] {
        if (n < 0 || (n > 0 && !partials)) throw Error{LZ_EINVAL, "bad partials buffer"};
        if (!nccl_comm) throw Error{LZ_EINVAL, "null NCCL communicator"};
        // ncclResult_t ncclAllReduce(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
        //                            ncclComm_t, cudaStream_t);  ncclDouble = 8, ncclSum = 0
        using AllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
        using ErrFn = const char* (*)(int);
        using AsyncErrFn = int (*)(void*, int*);
        static AllReduceFn all_reduce = nullptr;
        static ErrFn err_string = nullptr;
        static AsyncErrFn async_err = nullptr;
        static std::once_flag once;
        std::call_once(once, [] {
            // prefer the NCCL already mapped into the process (it created the communicator)
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return;
            all_reduce = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
            err_string = reinterpret_cast<ErrFn>(dlsym(h, "ncclGetErrorString"));
            async_err = reinterpret_cast<AsyncErrFn>(dlsym(h, "ncclCommGetAsyncError"));
        });
        if (!all_reduce) throw Error{LZ_ENCCL, "NCCL (libnccl.so.2) is not available in this process"};
        if (n == 0) return;
        constexpr int kInProgress = 7;  // ncclInProgress (non-blocking communicators)
        int rc = all_reduce(partials, partials, size_t(n), 8, 0, nccl_comm, (cudaStream_t)stream);
        // a non-blocking communicator enqueues in the background: wait until the collective is
        // on the stream, so the reduction kernel that follows is ordered after it
        while (rc == kInProgress && async_err) {
            int state = kInProgress;
            if (async_err(nccl_comm, &state) != 0) break;
            rc = state;
        }
        if (rc != 0)
            throw Error{LZ_ENCCL, std::string("ncclAllReduce: ") + (err_string ? err_string(rc) : std::to_string(rc))};
    });
}

int lz_fp64_peak(int device, double* tflops, double* ms_out) {
    return guarded([&] {
        DeviceGuard guard(device);
        int dev = 0, sms = 0;
        check_cuda(cudaGetDevice(&dev), "device");
        check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        const int threads = 256, blocks = sms * 8, iters = 2048;
        double* scratch = nullptr;
        check_cuda(cudaMalloc(&scratch, sizeof(double) * blocks), "malloc");
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        check_launch(lz::launch_probe(scratch, iters / 8, blocks, threads, 0), "probe", 0);  // warm-up
        cudaEventRecord(a, 0);
        check_launch(lz::launch_probe(scratch, iters, blocks, threads, 0), "probe", 0);
        cudaEventRecord(b, 0);
        check_cuda(cudaEventSynchronize(b), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(scratch);
        const double flops = 2.0 * 8.0 * 16.0 * double(iters) * double(threads) * double(blocks);
        *tflops = flops / (double(ms) * 1e-3) / 1e12;
        *ms_out = ms;
    });
}

}  // extern "C"
