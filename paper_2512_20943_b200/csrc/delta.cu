// Sparse-delta algebra and pruning-level bookkeeping on dense plane-major
// overlays (rows [width][ld] float64 + present u8 [n]).
//
//   k_compose        ss/model.py:294-311 compose_deltas (+ negate), n-way,
//                    one eps filter at the end
//   k_apply          ss/model.py:269-284 apply_delta, with the pruning-level
//                    selector of ss/pruning.py:79-90,111-113 folded in
//   k_quantize       ss/codec.py:193-199 encode_delta's quantisation rule and
//                    decode(encode(.)) values
//   prune ranks      ss/pruning.py:72-76 via compaction + stable radix sort
//   level sizes      ss/codec.py:200-207 exact GSDP size per pruning level
// All kernels stream the planes with unit stride across threads, two
// primitives per thread as 128-bit double2 accesses.
#include <algorithm>
#include <vector>

#include "context.h"
#include "scan_sort.cuh"

namespace airgs {

constexpr int kMaxCompose = 8;

struct ComposeArgs {
    const double *rows[kMaxCompose];
    const uint8_t *present[kMaxCompose];
    double sign[kMaxCompose];
    int nd;
};

// Two adjacent primitives (i, i+1; i even) per thread: every plane is read and
// written as 128-bit double2 (planes are 64-byte aligned, ld a multiple of 8,
// so i + 1 < ld always addresses the plane's padding at worst).  The padding
// lane (i + 1 >= n) is written as 0.
__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void st2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }
__device__ __forceinline__ uint32_t ld_u8x2(const uint8_t *p) {
    const uint16_t v = *reinterpret_cast<const uint16_t *>(p);
    return (uint32_t)v;
}

template <int W>
__global__ void __launch_bounds__(256)
k_compose(ComposeArgs a, int64_t n, int64_t ld, double eps, int apply_eps, double *__restrict__ out,
          uint8_t *__restrict__ outp) {
    const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    const bool two = i + 1 < n;
    double2 acc[W];
    bool any0 = false, any1 = false;
    for (int d = 0; d < a.nd; ++d) {
        const uint32_t pr = ld_u8x2(a.present[d] + i);
        const bool p0 = (pr & 0xffu) != 0, p1 = two && (pr >> 8) != 0;
        if (!p0 && !p1) continue;
        const double *r = a.rows[d] + i;
        const double s = a.sign[d];
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const double2 v = ld2(r + c * ld);
            // b.copy() / -b for the first present delta, acc + b afterwards
            if (p0) acc[c].x = any0 ? acc[c].x + s * v.x : s * v.x;
            if (p1) acc[c].y = any1 ? acc[c].y + s * v.y : s * v.y;
        }
        any0 |= p0;
        any1 |= p1;
    }
    bool keep0 = any0, keep1 = any1;
    if (apply_eps) {
        double m0 = 0.0, m1 = 0.0;
#pragma unroll
        for (int c = 0; c < W; ++c) {
            if (any0) m0 = fmax(m0, fabs(acc[c].x));
            if (any1) m1 = fmax(m1, fabs(acc[c].y));
        }
        keep0 = any0 && m0 > eps;
        keep1 = any1 && m1 > eps;
    }
    *reinterpret_cast<uint16_t *>(outp + i) = (uint16_t)((keep0 ? 1u : 0u) | (keep1 ? 0x100u : 0u));
#pragma unroll
    for (int c = 0; c < W; ++c)
        st2(out + c * ld + i, make_double2(keep0 ? acc[c].x : 0.0, keep1 ? acc[c].y : 0.0));
}

template <int W>
__global__ void __launch_bounds__(256)
k_apply(const double *__restrict__ canon, const double *__restrict__ ra, const uint8_t *__restrict__ pa,
        const uint8_t *__restrict__ sel, const int32_t *__restrict__ rank, int32_t kmin,
        const double *__restrict__ rb, const uint8_t *__restrict__ pb, int64_t n, int64_t ld,
        double *__restrict__ out) {
    const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    const bool two = i + 1 < n;
    const double *r[2] = {nullptr, nullptr};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t j = i + h;
        if (h && !two) break;
        const bool useA = (!sel || sel[j]) && (!rank || rank[j] >= kmin);
        if (useA) {
            if (ra && pa[j]) r[h] = ra;
        } else if (rb && pb[j]) {
            r[h] = rb;
        }
    }
    if (r[0] && r[0] == r[1]) {  // both rows from the same overlay: 128-bit loads
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const double2 cv = ld2(canon + c * ld + i), dv = ld2(r[0] + c * ld + i);
            st2(out + c * ld + i, make_double2(cv.x + dv.x, cv.y + dv.y));
        }
    } else {
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const double2 cv = ld2(canon + c * ld + i);
            const double x = r[0] ? cv.x + r[0][c * ld + i] : cv.x;
            const double y = !two ? 0.0 : r[1] ? cv.y + r[1][c * ld + i + 1] : cv.y;
            st2(out + c * ld + i, make_double2(x, y));
        }
    }
}

template <int W>
__global__ void __launch_bounds__(256)
k_quantize(const double *__restrict__ rows, const uint8_t *__restrict__ present, int64_t n, int64_t ld,
           double step, uint8_t *__restrict__ nz, double *__restrict__ deq, unsigned long long *bad) {
    const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    const uint32_t pr = ld_u8x2(present + i);
    const bool p0 = (pr & 0xffu) != 0, p1 = i + 1 < n && (pr >> 8) != 0;
    if (!p0 && !p1) {
        *reinterpret_cast<uint16_t *>(nz + i) = 0;
        return;
    }
    double2 q[W];
    bool any0 = false, any1 = false, over0 = false, over1 = false;
#pragma unroll
    for (int c = 0; c < W; ++c) {
        const double2 v = ld2(rows + c * ld + i);
        q[c] = make_double2(rint(v.x / step), rint(v.y / step));  // np.rint(v / quant_step): half-even
        any0 |= q[c].x != 0.0;
        any1 |= q[c].y != 0.0;
        over0 |= fabs(q[c].x) > 2147483647.0;
        over1 |= fabs(q[c].y) > 2147483647.0;
    }
    any0 &= p0;
    any1 &= p1;
    *reinterpret_cast<uint16_t *>(nz + i) = (uint16_t)((any0 ? 1u : 0u) | (any1 ? 0x100u : 0u));
    if (any0 && over0) atomicMin(bad, (unsigned long long)i);
    if (any1 && over1) atomicMin(bad, (unsigned long long)(i + 1));
    if (deq && (any0 || any1)) {
#pragma unroll
        for (int c = 0; c < W; ++c) {  // q.astype(f64) * quant_step
            double *o = deq + c * ld + i;
            if (any0 && any1) st2(o, make_double2(q[c].x * step, q[c].y * step));
            else if (any0) o[0] = q[c].x * step;
            else o[1] = q[c].y * step;
        }
    }
}

// --- prune ranks -------------------------------------------------------------

struct RevPresentIn {
    const uint8_t *present;
    int64_t n;
    __device__ int64_t operator()(int, int64_t j) const { return present[n - 1 - j] ? 1 : 0; }
};
struct RevPresentOut {
    const int64_t *usage;
    int64_t n;
    uint64_t *keys;
    uint32_t *vals;
    unsigned long long *umax;
    __device__ void operator()(int, int64_t j, int64_t ex, int64_t v) const {
        if (!v) return;
        const int64_t i = n - 1 - j;  // descending index order: ties prune higher index first
        const uint64_t u = (uint64_t)usage[i];
        keys[ex] = u;
        vals[ex] = (uint32_t)i;
        atomicMax(umax, (unsigned long long)u);
    }
};

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_scatter_rank(const uint32_t *__restrict__ vals, const int64_t *__restrict__ cnt,
                               int32_t *__restrict__ rank) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < *cnt) rank[vals[r]] = (int32_t)r;
}

// --- level sizes -------------------------------------------------------------

__device__ __forceinline__ int varint_len(int64_t v) {
    const int bits = v > 0 ? 64 - __clzll((long long)v) : 0;
    return bits <= 7 ? 1 : (bits + 6) / 7;
}

struct ChunkSummary {
    int64_t first, last, count, inner;
};

constexpr int kLvlThreads = 256, kLvlItems = 8, kLvlChunk = kLvlThreads * kLvlItems;

__global__ void __launch_bounds__(kLvlThreads)
k_level_chunks(const uint8_t *__restrict__ nz, const int32_t *__restrict__ rank, int64_t n,
               const int64_t *__restrict__ kmin, int nchunks, ChunkSummary *__restrict__ out) {
    const int l = blockIdx.y, c = blockIdx.x;
    const int64_t k = kmin[l];
    const int64_t lo = (int64_t)c * kLvlChunk + (int64_t)threadIdx.x * kLvlItems;
    int64_t first = -1, last = -1, cnt = 0, inner = 0;
    for (int t = 0; t < kLvlItems; ++t) {
        const int64_t i = lo + t;
        if (i >= n) break;
        if (nz[i] && (int64_t)rank[i] >= k) {
            if (last >= 0) inner += varint_len(i - last);
            else first = i;
            last = i;
            ++cnt;
        }
    }
    // exclusive max-scan of `last` across the block -> previous kept index
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t inc = last;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = max(inc, o);
    }
    __shared__ int64_t wmax[kLvlThreads / 32];
    __shared__ int64_t s_first[kLvlThreads / 32], s_cnt[kLvlThreads / 32], s_inner[kLvlThreads / 32];
    if (lane == 31) wmax[w] = inc;
    __syncthreads();
    int64_t before = -1;
    for (int ww = 0; ww < w; ++ww) before = max(before, wmax[ww]);
    int64_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) excl = -1;
    const int64_t prev = max(before, excl);
    if (first >= 0 && prev >= 0) inner += varint_len(first - prev);
    // block reductions: first kept (min over threads with data), count, inner
    int64_t f = first >= 0 ? first : INT64_MAX;
    for (int d = 16; d > 0; d >>= 1) {
        f = min(f, __shfl_down_sync(0xffffffffu, f, d));
        cnt += __shfl_down_sync(0xffffffffu, cnt, d);
        inner += __shfl_down_sync(0xffffffffu, inner, d);
    }
    if (lane == 0) {
        s_first[w] = f;
        s_cnt[w] = cnt;
        s_inner[w] = inner;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ChunkSummary s;
        s.first = INT64_MAX;
        s.count = 0;
        s.inner = 0;
        for (int ww = 0; ww < kLvlThreads / 32; ++ww) {
            s.first = min(s.first, s_first[ww]);
            s.count += s_cnt[ww];
            s.inner += s_inner[ww];
        }
        int64_t lst = -1;
        for (int ww = 0; ww < kLvlThreads / 32; ++ww) lst = max(lst, wmax[ww]);
        s.last = lst;
        out[(int64_t)l * nchunks + c] = s;
    }
}

__global__ void k_level_finish(const ChunkSummary *__restrict__ ch, int nchunks, int width,
                               int64_t *__restrict__ sizes) {
    const int l = blockIdx.x;
    if (threadIdx.x) return;
    int64_t prev = 0, total = 24, count = 0;  // encode_delta: prev = 0 before the first gap
    for (int c = 0; c < nchunks; ++c) {
        const ChunkSummary s = ch[(int64_t)l * nchunks + c];
        if (s.count == 0) continue;
        total += varint_len(s.first - prev) + s.inner;
        prev = s.last;
        count += s.count;
    }
    sizes[l] = total + 4 * (int64_t)width * count;
}

// --- host -------------------------------------------------------------------

template <template <int> class K, typename... Args>
static void launch_w(int W, dim3 g, dim3 b, cudaStream_t st, Args... args) {
    if (W == 17)
        K<17>::run(g, b, st, args...);
    else if (W == 26)
        K<26>::run(g, b, st, args...);
    else
        throw ApiFailure(AIRGS_E_STRUCTURAL, "no sh degree yields parameter width " + std::to_string(W));
}

template <int W>
struct ComposeK {
    template <typename... A>
    static void run(dim3 g, dim3 b, cudaStream_t st, A... a) { k_compose<W><<<g, b, 0, st>>>(a...); }
};
template <int W>
struct ApplyK {
    template <typename... A>
    static void run(dim3 g, dim3 b, cudaStream_t st, A... a) { k_apply<W><<<g, b, 0, st>>>(a...); }
};
template <int W>
struct QuantK {
    template <typename... A>
    static void run(dim3 g, dim3 b, cudaStream_t st, A... a) { k_quantize<W><<<g, b, 0, st>>>(a...); }
};

}  // namespace airgs

using namespace airgs;

extern "C" int airgs_delta_compose(airgs_ctx *ctx, int32_t ndeltas, const double *const *rows,
                                   const uint8_t *const *present, const double *signs, int64_t n, int32_t width,
                                   int64_t ld, double eps, int32_t apply_eps, double *out_rows,
                                   uint8_t *out_present, void *stream) {
    return guarded(ctx, [&] {
        if (ndeltas < 0 || ndeltas > kMaxCompose) throw ApiFailure(AIRGS_E_STRUCTURAL, "too many deltas to compose");
        if (n <= 0) return;
        ComposeArgs a;
        a.nd = ndeltas;
        for (int d = 0; d < ndeltas; ++d) {
            a.rows[d] = rows[d];
            a.present[d] = present[d];
            a.sign[d] = signs ? signs[d] : 1.0;
        }
        launch_w<ComposeK>(width, dim3((unsigned)ceil_div(n, 512)), dim3(256), (cudaStream_t)stream, a, n, ld, eps,
                           (int)apply_eps, out_rows, out_present);
        ++ctx->launches;
        check_launch();
    });
}

extern "C" int airgs_delta_apply(airgs_ctx *ctx, const double *canonical, const double *rows_a,
                                 const uint8_t *present_a, const uint8_t *sel_a, const int32_t *keep_rank,
                                 int32_t keep_min, const double *rows_b, const uint8_t *present_b, int64_t n,
                                 int32_t width, int64_t ld, double *params_out, void *stream) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        StageScope t0(ctx, (cudaStream_t)stream, kStageApply);
        launch_w<ApplyK>(width, dim3((unsigned)ceil_div(n, 512)), dim3(256), (cudaStream_t)stream, canonical, rows_a,
                         present_a, sel_a, keep_rank, keep_min, rows_b, present_b, n, ld, params_out);
        ++ctx->launches;
        check_launch();
        t0.end();
    });
}

extern "C" int airgs_quantize(airgs_ctx *ctx, const double *rows, const uint8_t *present, int64_t n, int32_t width,
                              int64_t ld, double step, uint8_t *nz_out, double *deq_out, int64_t *bad_index_out,
                              void *stream) {
    return guarded(ctx, [&] {
        if (!(step > 0.0)) throw ApiFailure(AIRGS_E_STRUCTURAL, "quant_step must be positive");
        if (bad_index_out) *bad_index_out = -1;
        if (n <= 0) return;
        cudaStream_t st = (cudaStream_t)stream;
        unsigned long long *bad = ctx->scratch_t<unsigned long long>(kSlotFlags, 2);
        const unsigned long long mx = ~0ull;
        h2d_small(ctx, bad, &mx, sizeof(mx), st);
        launch_w<QuantK>(width, dim3((unsigned)ceil_div(n, 512)), dim3(256), st, rows, present, n, ld, step, nz_out,
                         deq_out, bad);
        ++ctx->launches;
        check_launch();
        unsigned long long hb = 0;
        AIRGS_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        if (hb != ~0ull) {
            if (bad_index_out) *bad_index_out = (int64_t)hb;
            throw ApiFailure(AIRGS_E_STRUCTURAL,
                             "delta at " + std::to_string((long long)hb) + " overflows i32 fixed point");
        }
    });
}

extern "C" int airgs_prune_rank(airgs_ctx *ctx, const uint8_t *present, const int64_t *usage, int64_t n,
                                int32_t *rank_out, int64_t *count_out, void *stream) {
    return guarded(ctx, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        int64_t &L = ctx->launches;
        *count_out = 0;
        if (n <= 0) return;
        if (n > 0x7fffffffLL) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");
        uint64_t *keys = ctx->scratch_t<uint64_t>(kSlotKeys, n);
        uint32_t *vals = ctx->scratch_t<uint32_t>(kSlotVals, n);
        uint64_t *k2 = ctx->scratch_t<uint64_t>(kSlotKeysAlt, n);
        uint32_t *v2 = ctx->scratch_t<uint32_t>(kSlotValsAlt, n);
        int64_t *misc = ctx->scratch_t<int64_t>(kSlotMisc3, 8);
        int64_t *d_n = misc, *d_cnt = misc + 1;
        unsigned long long *umax = (unsigned long long *)(misc + 2);
        h2d_small(ctx, d_n, &n, sizeof(int64_t), st);
        AIRGS_CUDA_TRY(cudaMemsetAsync(umax, 0, sizeof(unsigned long long), st));
        const int bps = (int)std::max<int64_t>(1, ceil_div(n, kScanTile));
        int64_t *blocks = ctx->scratch_t<int64_t>(kSlotScanBlocks, bps);
        seg_scan<int64_t>(RevPresentIn{present, n}, RevPresentOut{usage, n, keys, vals, umax}, d_n, 1, n, blocks, d_cnt,
                          st, &L);
        check_launch();
        int64_t h[2];
        AIRGS_CUDA_TRY(cudaMemcpyAsync(h, d_cnt, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        const int64_t cnt = h[0];
        const uint64_t um = (uint64_t)h[1];
        k_fill_i32<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(rank_out, n, 0x7fffffff);
        ++L;
        if (cnt > 0) {
            int64_t *d_begin = misc + 3;
            AIRGS_CUDA_TRY(cudaMemsetAsync(d_begin, 0, sizeof(int64_t), st));
            const int nbits = bit_length(um);
            const uint32_t *sv = vals;
            if (nbits > 0) {
                uint32_t *hist = ctx->scratch_t<uint32_t>(kSlotHist, (size_t)256 * ceil_div(cnt, kSortTile));
                bool alt = radix_sort<uint64_t>(keys, vals, k2, v2, d_begin, d_cnt, 1, cnt, nbits, hist, st, &L);
                if (alt) sv = v2;
            }
            k_scatter_rank<<<(unsigned)ceil_div(cnt, 256), 256, 0, st>>>(sv, d_cnt, rank_out);
            ++L;
        }
        check_launch();
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        *count_out = cnt;
    });
}

extern "C" int airgs_level_sizes(airgs_ctx *ctx, const uint8_t *nz, const int32_t *rank, int64_t n, int32_t width,
                                 const int64_t *kmin, int32_t nlevels, int64_t *sizes_out, void *stream) {
    return guarded(ctx, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        if (nlevels <= 0) return;
        if (n <= 0) {
            for (int l = 0; l < nlevels; ++l) sizes_out[l] = 24;
            return;
        }
        const int nchunks = (int)ceil_div(n, kLvlChunk);
        int64_t *d_k = ctx->scratch_t<int64_t>(kSlotMisc2, (size_t)2 * nlevels);
        int64_t *d_sizes = d_k + nlevels;
        ChunkSummary *ch = (ChunkSummary *)ctx->scratch(kSlotMisc1, sizeof(ChunkSummary) * (size_t)nchunks * nlevels);
        h2d_small(ctx, d_k, kmin, sizeof(int64_t) * nlevels, st);
        k_level_chunks<<<dim3((unsigned)nchunks, (unsigned)nlevels), kLvlThreads, 0, st>>>(nz, rank, n, d_k, nchunks, ch);
        k_level_finish<<<nlevels, 32, 0, st>>>(ch, nchunks, width, d_sizes);
        ctx->launches += 2;
        check_launch();
        AIRGS_CUDA_TRY(cudaMemcpyAsync(sizes_out, d_sizes, sizeof(int64_t) * nlevels, cudaMemcpyDeviceToHost, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    });
}
