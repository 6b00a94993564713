// Segmented scans and a stable segmented LSD radix sort, hand-written with
// warp-level primitives (shuffles, match_any, ballots).  No CUB.
//
// Segment layout used by every primitive: nseg segments, segment s owns
// elements [begin[s], begin[s] + count[s]) of the data arrays; the host
// passes an upper bound `maxc` on count[] so the grid is fixed at
// nseg * blocks_per_seg and surplus blocks exit (no device->host sync needed
// to size a launch).
#pragma once

#include "common.cuh"

namespace airgs {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;                       // per thread
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048 elements per block

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;                      // 256 keys per round
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 keys per block
constexpr int kSortWarps = kSortThreads / 32;

// ---------------------------------------------------------------------------
// warp / block scans

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    return v;
}

// Exclusive scan of one value per thread over a block of NT threads.
// Returns the exclusive prefix; *total receives the block sum.
template <typename T, int NT>
__device__ __forceinline__ T block_exclusive_scan(T v, T *total) {
    __shared__ T warp_tot[NT / 32 + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        T t = lane < NT / 32 ? warp_tot[lane] : T(0);
        T ti = warp_inclusive_scan(t);
        if (lane < NT / 32) warp_tot[lane] = ti - t;  // exclusive warp offsets
        if (lane == NT / 32 - 1) warp_tot[NT / 32] = ti;  // block total
    }
    __syncthreads();
    T res = warp_tot[w] + inc - v;
    *total = warp_tot[NT / 32];
    __syncthreads();  // warp_tot is reused by the next call
    return res;
}

// ---------------------------------------------------------------------------
// segmented exclusive scan driven by functors
//   In:  T operator()(int seg, int64_t i) const        value of element i of seg
//   Out: void operator()(int seg, int64_t i, T excl, T v) const

template <typename T, typename In>
__global__ void __launch_bounds__(kScanThreads)
k_seg_scan_reduce(In in, const int64_t *__restrict__ count, int bps, T *__restrict__ block_sums) {
    const int seg = blockIdx.x / bps, b = blockIdx.x % bps;
    const int64_t n = count[seg];
    const int64_t lo = (int64_t)b * kScanTile;
    T s = 0;
    if (lo < n) {
        for (int k = 0; k < kScanItems; ++k) {
            int64_t i = lo + (int64_t)k * kScanThreads + threadIdx.x;
            if (i < n) s += in(seg, i);
        }
    }
    s = warp_reduce_sum(s);
    __shared__ T wt[kScanThreads / 32];
    if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += wt[w];
        block_sums[blockIdx.x] = t;
    }
}

// one block per segment: exclusive scan of its bps block sums (in place),
// segment total to seg_total[seg] (optional)
template <typename T>
__global__ void __launch_bounds__(1024)
k_seg_scan_blocks(T *__restrict__ block_sums, int bps, T *__restrict__ seg_total) {
    const int seg = blockIdx.x;
    T *p = block_sums + (int64_t)seg * bps;
    T carry = 0;
    for (int base = 0; base < bps; base += 1024) {
        int i = base + threadIdx.x;
        T v = i < bps ? p[i] : T(0);
        T tot;
        T ex = block_exclusive_scan<T, 1024>(v, &tot);
        if (i < bps) p[i] = carry + ex;
        carry += tot;
    }
    if (seg_total && threadIdx.x == 0) seg_total[seg] = carry;
}

template <typename T, typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads)
k_seg_scan_apply(In in, Out out, const int64_t *__restrict__ count, int bps,
                 const T *__restrict__ block_off) {
    const int seg = blockIdx.x / bps, b = blockIdx.x % bps;
    const int64_t n = count[seg];
    const int64_t lo = (int64_t)b * kScanTile;
    if (lo >= n) return;  // uniform per block
    // blocked arrangement: thread t owns elements lo + t*kScanItems + k
    T v[kScanItems];
    T local = 0;
    const int64_t mine = lo + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = mine + k;
        v[k] = i < n ? in(seg, i) : T(0);
        local += v[k];
    }
    T tot;
    T ex = block_exclusive_scan<T, kScanThreads>(local, &tot) + block_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = mine + k;
        if (i < n) out(seg, i, ex, v[k]);
        ex += v[k];
    }
}

// Host driver.  block_sums must hold nseg*bps elements; seg_total nseg (or null).
template <typename T, typename In, typename Out>
void seg_scan(In in, Out out, const int64_t *count, int nseg, int64_t maxc, T *block_sums,
              T *seg_total, cudaStream_t st, int64_t *launches) {
    if (nseg <= 0) return;
    int bps = (int)std::max<int64_t>(1, ceil_div(maxc, kScanTile));
    dim3 grid((unsigned)(nseg * bps));
    k_seg_scan_reduce<T, In><<<grid, kScanThreads, 0, st>>>(in, count, bps, block_sums);
    k_seg_scan_blocks<T><<<nseg, 1024, 0, st>>>(block_sums, bps, seg_total);
    k_seg_scan_apply<T, In, Out><<<grid, kScanThreads, 0, st>>>(in, out, count, bps, block_sums);
    *launches += 3;
}

// ---------------------------------------------------------------------------
// stable segmented LSD radix sort (keys KeyT, values uint32)

template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const KeyT *__restrict__ keys, const int64_t *__restrict__ begin,
             const int64_t *__restrict__ count, int bps, int shift, int dbits,
             uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    const int seg = blockIdx.x / bps, b = blockIdx.x % bps;
    const int radix = 1 << dbits;
    for (int d = threadIdx.x; d < radix; d += kSortThreads) h[d] = 0;
    __syncthreads();
    const int64_t n = count[seg], lo = (int64_t)b * kSortTile;
    const KeyT *kp = keys + begin[seg];
    if (lo < n) {
        const int64_t hi = min(n, lo + (int64_t)kSortTile);
        for (int64_t i = lo + threadIdx.x; i < hi; i += kSortThreads) {
            uint32_t d = (uint32_t)(kp[i] >> shift) & (uint32_t)(radix - 1);
            atomicAdd(&h[d], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kSortThreads)
        hist[((int64_t)seg * radix + d) * bps + b] = h[d];
}

// per segment exclusive scan of radix*bps counters (digit-major)
static __global__ void __launch_bounds__(1024)
k_radix_scan(uint32_t *__restrict__ hist, int bps, int radix) {
    const int seg = blockIdx.x;
    uint32_t *p = hist + (int64_t)seg * radix * bps;
    const int64_t m = (int64_t)radix * bps;
    uint32_t carry = 0;
    for (int64_t base = 0; base < m; base += 1024) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < m ? p[i] : 0u;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan<uint32_t, 1024>(v, &tot);
        if (i < m) p[i] = carry + ex;
        carry += tot;
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const KeyT *__restrict__ kin, const uint32_t *__restrict__ vin,
                KeyT *__restrict__ kout, uint32_t *__restrict__ vout,
                const int64_t *__restrict__ begin, const int64_t *__restrict__ count, int bps,
                int shift, int dbits, const uint32_t *__restrict__ offs) {
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[kSortWarps][256];
    const int seg = blockIdx.x / bps, b = blockIdx.x % bps;
    const int radix = 1 << dbits;
    const int64_t n = count[seg], lo = (int64_t)b * kSortTile;
    if (lo >= n) return;
    const int64_t hi = min(n, lo + (int64_t)kSortTile);
    const int64_t bg = begin[seg];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < radix; d += kSortThreads)
        run[d] = offs[((int64_t)seg * radix + d) * bps + b];
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = lo; base < hi; base += kSortThreads) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < hi;
        KeyT key = valid ? kin[bg + i] : KeyT(0);
        uint32_t val = valid ? vin[bg + i] : 0u;
        uint32_t dig = valid ? ((uint32_t)(key >> shift) & (uint32_t)(radix - 1)) : 0xffffffffu;
        for (int d = lane; d < radix; d += 32) wcnt[w][d] = 0;
        __syncthreads();
        unsigned peers = __match_any_sync(0xffffffffu, dig);
        int rank_in_warp = __popc(peers & lt);
        if (valid && rank_in_warp == 0) wcnt[w][dig] = __popc(peers);
        __syncthreads();
        // per digit: running offset + exclusive scan over warps
        for (int d = threadIdx.x; d < radix; d += kSortThreads) {
            uint32_t s = run[d];
#pragma unroll
            for (int ww = 0; ww < kSortWarps; ++ww) {
                uint32_t c = wcnt[ww][d];
                wcnt[ww][d] = s;
                s += c;
            }
            run[d] = s;
        }
        __syncthreads();
        if (valid) {
            uint32_t pos = wcnt[w][dig] + (uint32_t)rank_in_warp;
            kout[bg + pos] = key;
            vout[bg + pos] = val;
        }
        __syncthreads();
    }
}

// Sort (keys, vals) in place per segment by bits [0, nbits) of the key.
// Ping-pongs through (kalt, valt); returns true if the result is in the alt
// buffers.  hist must hold nseg*256*bps uint32.
template <typename KeyT>
bool radix_sort(KeyT *keys, uint32_t *vals, KeyT *kalt, uint32_t *valt, const int64_t *begin,
                const int64_t *count, int nseg, int64_t maxc, int nbits, uint32_t *hist,
                cudaStream_t st, int64_t *launches) {
    if (nseg <= 0 || maxc <= 0 || nbits <= 0) return false;
    const int bps = (int)ceil_div(maxc, kSortTile);
    const dim3 grid((unsigned)(nseg * bps));
    bool alt = false;
    for (int shift = 0; shift < nbits; shift += 8) {
        const int dbits = std::min(8, nbits - shift);
        const KeyT *ki = alt ? kalt : keys;
        const uint32_t *vi = alt ? valt : vals;
        KeyT *ko = alt ? keys : kalt;
        uint32_t *vo = alt ? vals : valt;
        k_radix_hist<KeyT><<<grid, kSortThreads, 0, st>>>(ki, begin, count, bps, shift, dbits, hist);
        k_radix_scan<<<nseg, 1024, 0, st>>>(hist, bps, 1 << dbits);
        k_radix_scatter<KeyT><<<grid, kSortThreads, 0, st>>>(ki, vi, ko, vo, begin, count, bps, shift,
                                                             dbits, hist);
        *launches += 3;
        alt = !alt;
    }
    return alt;
}

}  // namespace airgs
