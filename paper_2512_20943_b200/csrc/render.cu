// Batched rasterizer for the AirGS evaluation path on B200 (sm_100a).
//
// Pipeline per batch of view items (frame, camera):
//   k_project       fp64 activation + EWA projection, op-for-op with
//                   ss/rasterizer.py:100-212 (one thread per primitive, all
//                   views of its frame in the inner loop so the parameter row
//                   and the view-independent activation are read/computed once);
//                   emits a 96-byte record, an orderable depth key, and a
//                   per-tile histogram (atomics)
//   tile scan       exclusive scan of the histogram (warp scans) -> tile ranges
//   k_emit          primitive ids into their tiles' ranges (atomic cursors, any order)
//   k_composite     16x16 tile per CTA: the tile's list is sorted in shared memory
//                   by (depth key, primitive index) -- exactly the reference's
//                   stable argsort order restricted to the tile -- then
//                   composited front to back with exact early termination; fp32
//                   log2-domain candidate pass with a proven guard band, exact
//                   fp64 replay of _composite.pyx:42-73 for candidates; fused
//                   usage counts and per-warp SSE partials
//   k_sse_items     deterministic per-item SSE reduction
// Tiles whose list exceeds the in-shared-memory sort capacity are sorted
// beforehand by a segmented radix sort over (index, then depth key).
#include <algorithm>
#include <cstring>
#include <cmath>
#include <type_traits>
#include <vector>

#include <cub/block/block_radix_sort.cuh>

#include "context.h"
#include "exp_table.h"
#include "scan_sort.cuh"

namespace airgs {

// ---------------------------------------------------------------------------
// projection

// ellipse-vs-tile cull record of a (view, primitive) (see make_cull_rec)
constexpr uint32_t kCullFlag = 0x80000000u;
struct __align__(16) CullRec {
    float A, B, C, rX;    // 0.5 a, b, 0.5 c (fp32); 1 / (2 C)
    float rY, mx, my, t;  // 1 / (2 A); mean - 0.5 relative to the range's first pixel; t (fp32)
};

struct ProjArgs {
    const airgs_frame *frames;
    const airgs_camera *cams;
    const int32_t *frame_item_ptr;  // CSR over frames
    const int32_t *frame_items;
    const int32_t *item_cam;
    const int64_t *tile_base;  // [nitems] first global tile of each item
    const int32_t *tiles_x;    // [nitems]
    Rec *recs;                 // [nitems][stride]
    uint64_t *depth;           // [nitems][stride] orderable depth keys
    int32_t *ntiles;           // [nitems][stride] tiles touched (0 = empty bbox, -1 = no tile)
    uint2 *binrec;             // [nitems][stride] tile range u0 | u1 << 16 (| kCullFlag), v0 | v1 << 16 (when ntiles > 0)
    CullRec *cullrec;          // [nitems][stride] (flagged ranges only)
    unsigned int *flags;
    int64_t stride;
    unsigned long long *stats;  // diagnostic decision margins (null: off)
    const int64_t *const *item_frozen;  // per item: frozen order positions or null (null: none at all)
};

// Compositing-order key of a kept primitive: its position in a frozen order
// (< 2^63, ahead of everything else) or, for primitives outside it and in the
// unfrozen case, the orderable depth key (>= 2^63 for z > 0); ties in either
// resolve by index (ss/rasterizer.py:127-142, stable argsorts).
__device__ __forceinline__ unsigned long long order_key_of(const int64_t *frozen, int64_t i, double tz);


__device__ __forceinline__ double dist_to_int(double x) { return fabs(x - rint(x)); }

__device__ __forceinline__ void margin_min(unsigned long long *stats, int slot, double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) b = min(b, __shfl_xor_sync(0xffffffffu, b, d));
    if ((threadIdx.x & 31) == 0) atomicMin(stats + slot, b);
}

__device__ __forceinline__ double dot3_blas(double x0, double x1, double x2, double y0, double y1,
                                            double y2) {
    // OpenBLAS accumulation order of every small matmul in _prepare
    return fma(x2, y2, fma(x1, y1, x0 * y0));
}

__device__ __forceinline__ double sigmoid_ref(double x) {
    return 0.5 * (1.0 + tanh(0.5 * x));  // ss/model.py:63-64
}

// Orderable 64-bit key of a double (monotone for all finite values).
__device__ __forceinline__ unsigned long long order_key(double z) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(z);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// 32-bit list-entry key, monotone in the 64-bit order key: frozen positions
// and the seam's input indices (< 2^30) first, then negative depths (a
// near_clip < 0 camera keeps near_clip < z <= 0, ss/rasterizer.py:126), then
// positive depths; fp32 depth bits (ties between distinct 64-bit keys are
// resolved by the tile sort's exact-key run fix)
__device__ __forceinline__ uint32_t list_key32(unsigned long long zk) {
    if (zk >> 63) return 0x80000000u | (__float_as_uint((float)__longlong_as_double((long long)(zk & 0x7fffffffffffffffull))) >> 1);
    if (zk < (1ull << 30)) return (uint32_t)zk;
    const float f = (float)__longlong_as_double((long long)~zk);  // z <= -0
    return 0x40000000u | (~__float_as_uint(f) >> 1);
}

__device__ __forceinline__ unsigned long long order_key_of(const int64_t *frozen, int64_t i, double tz) {
    if (frozen && frozen[i] >= 0) return (unsigned long long)frozen[i];
    return order_key(tz);
}

// Tile range of a record: clipped bbox intersected with the pixel centres
// inside the threshold-ellipse AABB (|dx| <= hx, |dy| <= hy); pixels outside
// cannot pass the weight test, so tiles outside this range are never needed.
__device__ __forceinline__ bool rec_tile_range(const Rec &r, int &u0, int &u1, int &v0, int &v1) {
    int xa = r.x0, xb = r.x1 - 1, ya = r.y0, yb = r.y1 - 1;
    if (r.hx < 1e29f) {
        xa = max(xa, (int)ceilf((float)(r.mx - 0.5) - r.hx));
        xb = min(xb, (int)floorf((float)(r.mx - 0.5) + r.hx));
    }
    if (r.hy < 1e29f) {
        ya = max(ya, (int)ceilf((float)(r.my - 0.5) - r.hy));
        yb = min(yb, (int)floorf((float)(r.my - 0.5) + r.hy));
    }
    if (xa > xb || ya > yb) return false;
    u0 = xa / kTile;
    u1 = xb / kTile;
    v0 = ya / kTile;
    v1 = yb / kTile;
    return true;
}

// Ellipse-vs-tile cull of the binning.  For a primitive-view whose tile range
// spans 2..4 tiles in both directions (the corners of its threshold AABB are
// where tiles can miss the ellipse) the projection stores the fp32 inputs of
// the test in a 32-byte cull record and flags the range (bit 31 of binrec.x);
// the binning then drops a (primitive, tile) pair when a conservative lower
// bound of e = 0.5 (a dx^2 + c dy^2) + b dx dy over the tile's pixel centres
// exceeds t = ln(al / EPS) (+ pad): no pixel of that tile can pass the weight
// test.  The tests run in the binning, where (primitive, tile) pairs are dealt
// evenly over the warp's lanes.  oracle/airgs_oracle.py restates it op for op.
#ifndef TILE_CULL
#define TILE_CULL 1
#endif

// Lower bound (conservative by 1e-4 of the terms' magnitude + 1e-3, far above
// fp32 rounding) of min Q(dx, dy) = A dx^2 + B dx dy + C dy^2 over the
// rectangle [x0, x1] x [y0, y1] (A, C > 0, positive definite): 0 if the
// rectangle holds the origin, else the smallest of the four edges' minima,
// each the 1-D quadratic at its clamped vertex (vertices from the reciprocals
// rX = 1/(2C), rY = 1/(2A); evaluating a rounded vertex only raises the value
// by Q delta^2, far inside the slack).  Plain fp32 (-fmad=false).
__device__ __forceinline__ float quad_rect_min_lb(float A, float B, float C, float rX, float rY, float x0, float x1,
                                                  float y0, float y1) {
    if (x0 <= 0.0f && x1 >= 0.0f && y0 <= 0.0f && y1 >= 0.0f) return 0.0f;
    auto edge = [B](float P, float Q, float r, float X, float lo, float hi) {
        // min over t in [lo, hi] of P X^2 + B X t + Q t^2
        const float t = fminf(fmaxf(-B * X * r, lo), hi);
        const float a = P * X * X, b = B * X * t, c = Q * t * t;
        return (a + b + c) - (1e-4f * (a + fabsf(b) + c) + 1e-3f);
    };
    const float ex = fminf(edge(A, C, rX, x0, y0, y1), edge(A, C, rX, x1, y0, y1));
    const float ey = fminf(edge(C, A, rY, y0, x0, x1), edge(C, A, rY, y1, x0, x1));
    return fminf(ex, ey);
}

// may the ellipse of cull record c reach tile (du, dv) of its range?
__device__ __forceinline__ bool cull_keep(const CullRec &c, int du, int dv) {
    const float x0 = (float)(du * kTile) - c.mx, x1 = (float)(du * kTile + kTile - 1) - c.mx;
    const float y0 = (float)(dv * kTile) - c.my, y1 = (float)(dv * kTile + kTile - 1) - c.my;
    return !(quad_rect_min_lb(c.A, c.B, c.C, c.rX, c.rY, x0, x1, y0, y1) > c.t);
}

// the cull record of a projected record with tile range (u0..u1, v0..v1), or false
__device__ __forceinline__ bool make_cull_rec(const Rec &r, int u0, int u1, int v0, int v1, double t, CullRec &c) {
    const int nu = u1 - u0 + 1, nv = v1 - v0 + 1;
    if (!TILE_CULL || nu < 2 || nv < 2 || nu > 4 || nv > 4 || !(r.hx < 1e29f && r.hy < 1e29f)) return false;
    c.A = (float)(0.5 * r.ca);
    c.B = (float)r.cb;
    c.C = (float)(0.5 * r.cc);
    if (!(c.A > 0.0f && c.C > 0.0f)) return false;
    c.rX = 1.0f / (2.0f * c.C);
    c.rY = 1.0f / (2.0f * c.A);
    c.mx = (float)(r.mx - (double)(u0 * kTile)) - 0.5f;
    c.my = (float)(r.my - (double)(v0 * kTile)) - 0.5f;
    c.t = (float)t;
    return true;
}

constexpr int kProjThreads = 128;
#ifndef PROJ_MIN_BLOCKS
#define PROJ_MIN_BLOCKS 4
#endif
#ifndef PROJ_STAGE_REC
#define PROJ_STAGE_REC 1
#endif

// WMAX = 17 when every frame of the launch is SH degree 0 (fewer live registers),
// 26 otherwise (handles both widths).
template <int WMAX>
__global__ void __launch_bounds__(kProjThreads, PROJ_MIN_BLOCKS) k_project(ProjArgs a) {
    const int f = blockIdx.y;
    const airgs_frame fr = a.frames[f];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ib = a.frame_item_ptr[f], ie = a.frame_item_ptr[f + 1];
    if (ib == ie || (int64_t)blockIdx.x * blockDim.x >= fr.count) return;  // block-uniform
    const bool active = i < fr.count;
    const int64_t ld = fr.ld;
    const int W = fr.width;
    double p[26];
#pragma unroll
    for (int c = 0; c < 26; ++c) p[c] = (active && c < W && c < WMAX) ? fr.params[i + c * ld] : 0.0;

    // _activate (ss/rasterizer.py:100-110)
    const double qn = sqrt(((p[3] * p[3] + p[4] * p[4]) + p[5] * p[5]) + p[6] * p[6]);
    bool finite = true;
#pragma unroll
    for (int c = 0; c < WMAX; ++c) finite &= isfinite(p[c]);
    const bool valid = active && qn != 0.0 && finite;
    if (active && !valid) atomicOr(a.flags, (unsigned)kFlagInvalidParam);
    const double w_ = p[3] / qn, x_ = p[4] / qn, y_ = p[5] / qn, z_ = p[6] / qn;
    const double s0 = exp(2.0 * p[7]), s1 = exp(2.0 * p[8]), s2 = exp(2.0 * p[9]);
    const double alpha = sigmoid_ref(p[10]);
    // quat_to_matrix (ss/model.py:72-85), elementwise, no fusion
    double m[9];
    m[0] = 1.0 - 2.0 * (y_ * y_ + z_ * z_);
    m[1] = 2.0 * (x_ * y_ - w_ * z_);
    m[2] = 2.0 * (x_ * z_ + w_ * y_);
    m[3] = 2.0 * (x_ * y_ + w_ * z_);
    m[4] = 1.0 - 2.0 * (x_ * x_ + z_ * z_);
    m[5] = 2.0 * (y_ * z_ - w_ * x_);
    m[6] = 2.0 * (x_ * z_ - w_ * y_);
    m[7] = 2.0 * (y_ * z_ + w_ * x_);
    m[8] = 1.0 - 2.0 * (x_ * x_ + y_ * y_);
    // cov3d = (R * s2) @ R^T  (ss/rasterizer.py:159), full 3x3 (not symmetric in fp)
    double cv[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            cv[3 * r + c] = dot3_blas(m[3 * r] * s0, m[3 * r + 1] * s1, m[3 * r + 2] * s2, m[3 * c], m[3 * c + 1],
                                      m[3 * c + 2]);
    const bool live = valid && alpha > kEpsContrib;
    // threshold-ellipse extent factor 2 max(t, 0), t = ln(al / EPS) (+ outward pad): per primitive
    const double t2 = live ? 2.0 * fmax(log(alpha / kEpsContrib) * 1.0002 + 2e-4, 0.0) : 0.0;
    // SH degree 0: colour is view independent -- compute once
    double col0[3] = {0.0, 0.0, 0.0};
    if (W == 17 && live) {
        col0[0] = sigmoid_ref(p[11] + kShC0 * p[14]);
        col0[1] = sigmoid_ref(p[12] + kShC0 * p[15]);
        col0[2] = sigmoid_ref(p[13] + kShC0 * p[16]);
    }
    // the frame's cameras, staged in shared memory a chunk at a time: the view
    // loop then reads them as broadcasts instead of dependent global loads
    constexpr int kCamStage = 32;
    constexpr int kCamWords = (int)(sizeof(airgs_camera) / 8);
    __shared__ unsigned long long scam_raw[kCamStage * kCamWords];
    __shared__ int sitem[kCamStage];
    const airgs_camera *scam = reinterpret_cast<const airgs_camera *>(scam_raw);
    __shared__ Rec srec[PROJ_STAGE_REC ? kProjThreads : 1];
    for (int cb = ib; cb < ie; cb += kCamStage) {
        const int ncb = min(kCamStage, ie - cb);
        __syncthreads();  // the previous chunk is consumed
        for (int k = threadIdx.x; k < ncb * kCamWords; k += kProjThreads) {
            const int q = k / kCamWords, wd = k - q * kCamWords;
            const int item = a.frame_items[cb + q];
            scam_raw[k] = reinterpret_cast<const unsigned long long *>(a.cams + a.item_cam[item])[wd];
            if (wd == 0) sitem[q] = item;
        }
        __syncthreads();
    for (int q = 0; q < ncb; ++q) {
        const int item = sitem[q];
        const int64_t o = (int64_t)item * a.stride + i;
        const airgs_camera &cam = scam[q];
        const double *R = cam.rot;
        bool need = false;
        int nt = 0;
        double tz = 0.0;
        double bbm = 1.0;  // stats: bbox floor/ceil argument margin
        if (live) tz = dot3_blas(p[0], p[1], p[2], R[6], R[7], R[8]) + cam.trans[2];
        if (a.stats) margin_min(a.stats, kMarginNear, live ? fabs(tz - cam.near_clip) : 1e300);
        if (live && tz > cam.near_clip) {
            const double tx = dot3_blas(p[0], p[1], p[2], R[0], R[1], R[2]) + cam.trans[0];
            const double ty = dot3_blas(p[0], p[1], p[2], R[3], R[4], R[5]) + cam.trans[1];
            const double fl = cam.focal;
            const double mx = fl * tx / tz + 0.5 * (double)cam.width;
            const double my = fl * ty / tz + 0.5 * (double)cam.height;
            // J (2x3) @ R_wc with the reference's explicit zeros
            const double j00 = fl / tz;
            const double zz = tz * tz;
            const double j02 = -fl * tx / zz;
            const double j12 = -fl * ty / zz;
            double M[6];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                M[c] = dot3_blas(j00, 0.0, j02, R[c], R[3 + c], R[6 + c]);
                M[3 + c] = dot3_blas(0.0, j00, j12, R[c], R[3 + c], R[6 + c]);
            }
            double MC[6];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    MC[3 * r + c] = dot3_blas(M[3 * r], M[3 * r + 1], M[3 * r + 2], cv[c], cv[3 + c], cv[6 + c]);
            const double a2 = dot3_blas(MC[0], MC[1], MC[2], M[0], M[1], M[2]) + kCovBlur;
            const double b2 = dot3_blas(MC[0], MC[1], MC[2], M[3], M[4], M[5]);
            const double c2 = dot3_blas(MC[3], MC[4], MC[5], M[3], M[4], M[5]) + kCovBlur;
            const double det = a2 * c2 - b2 * b2;
            Rec rec;
            rec.mx = mx;
            rec.my = my;
            rec.ca = c2 / det;
            rec.cb = -b2 / det;
            rec.cc = a2 / det;
            const double dd = a2 - c2;
            const double eig = 0.5 * (a2 + c2) + sqrt(fmax(0.25 * (dd * dd) + b2 * b2, 0.0));
            const double rad = kRadiusSigma * sqrt(eig);
            const double Wd = (double)cam.width, Hd = (double)cam.height;
            if (a.stats)
                bbm = fmin(bbm, fmin(fmin(dist_to_int(mx - rad), dist_to_int(mx + rad)),
                                     fmin(dist_to_int(my - rad), dist_to_int(my + rad))));
            rec.x0 = (int32_t)fmin(fmax(floor(mx - rad), 0.0), Wd);
            rec.x1 = (int32_t)fmin(fmax(ceil(mx + rad) + 1.0, 0.0), Wd);
            rec.y0 = (int32_t)fmin(fmax(floor(my - rad), 0.0), Hd);
            rec.y1 = (int32_t)fmin(fmax(ceil(my + rad) + 1.0, 0.0), Hd);
            if (WMAX == 26 && W == 26) {  // colour (ss/rasterizer.py:183-198), view dependent
                const double d0 = p[0] - cam.center[0], d1 = p[1] - cam.center[1], d2 = p[2] - cam.center[2];
                double dn = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
                if (dn == 0.0) dn = 1.0;
                const double h0 = d0 / dn, h1 = d1 / dn, h2 = d2 / dn;
                rec.cr = sigmoid_ref((p[11] + kShC0 * p[14]) + kShC1 * ((-h1 * p[17] + h2 * p[20]) - h0 * p[23]));
                rec.cg = sigmoid_ref((p[12] + kShC0 * p[15]) + kShC1 * ((-h1 * p[18] + h2 * p[21]) - h0 * p[24]));
                rec.cbl = sigmoid_ref((p[13] + kShC0 * p[16]) + kShC1 * ((-h1 * p[19] + h2 * p[22]) - h0 * p[25]));
            } else {
                rec.cr = col0[0];
                rec.cg = col0[1];
                rec.cbl = col0[2];
            }
            rec.al = alpha;
            {
                // e >= dx^2 / (2 Sxx) with Sigma = cov2d, so |dx| > sqrt(2 t Sxx) => e > t
                // (t2 = 2 max(t, 0), t = ln(al/EPS) padded: view independent, hoisted)
                const double hx = sqrt(t2 * (a2 + 1e-9 * a2)) * 1.0002 + 1e-3;
                const double hy = sqrt(t2 * (c2 + 1e-9 * c2)) * 1.0002 + 1e-3;
                rec.hx = det > 0.0 && isfinite(hx) ? (float)hx * 1.0001f : 1e30f;
                rec.hy = det > 0.0 && isfinite(hy) ? (float)hy * 1.0001f : 1e30f;
            }
            int u0, u1, v0, v1;
            const bool has_bbox = rec.x1 > rec.x0 && rec.y1 > rec.y0;
            if (has_bbox && rec_tile_range(rec, u0, u1, v0, v1)) {
                nt = (u1 - u0 + 1) * (v1 - v0 + 1);
                CullRec cr;
                const bool cull = a.cullrec && make_cull_rec(rec, u0, u1, v0, v1, 0.5 * t2, cr);
                if (cull) a.cullrec[o] = cr;
                a.binrec[o] = make_uint2((uint32_t)u0 | ((uint32_t)u1 << 16) | (cull ? kCullFlag : 0u),
                                         (uint32_t)v0 | ((uint32_t)v1 << 16));
            }
            const int64_t *fz = a.item_frozen ? a.item_frozen[item] : nullptr;
            const unsigned long long zk = order_key_of(fz, i, tz);
            // records of primitives that reach no tile are read only by the diagnostic counters
            need = nt > 0 || (has_bbox && a.stats);
            if (need) {
                if (PROJ_STAGE_REC)
                    srec[threadIdx.x] = rec;
                else
                    a.recs[o] = rec;
                a.depth[o] = zk;
            }
            if (nt <= 0 && has_bbox) nt = -1;  // evaluated by the reference, but no pixel can pass the weight test
        }
        if (active) a.ntiles[o] = nt;
        if (a.stats) margin_min(a.stats, kMarginBBox, bbm);
        if (a.stats) {
            const unsigned nm = __ballot_sync(0xffffffffu, need && nt > 0);
            if ((threadIdx.x & 31) == 0 && nm) atomicAdd(a.stats + kStatRecords, (unsigned long long)__popc(nm));
        }
        if (PROJ_STAGE_REC) {
            // the warp's 32 records leave as contiguous 16-byte chunks (each store
            // instruction writes 512 consecutive bytes instead of 32 scattered pieces)
            const unsigned needm = __ballot_sync(0xffffffffu, need);
            if (needm) {
                __syncwarp();
                const int lane = threadIdx.x & 31;
                const float4 *src = reinterpret_cast<const float4 *>(srec + (threadIdx.x & ~31));
                float4 *dst = reinterpret_cast<float4 *>(a.recs + (o - lane));
                constexpr int kChunks = (int)(sizeof(Rec) / 16);
#pragma unroll
                for (int k = 0; k < kChunks; ++k) {
                    const int c = k * 32 + lane;
                    if ((needm >> (c / kChunks)) & 1u) dst[c] = src[c];
                }
                __syncwarp();
            }
        }
    }
    }
    if (a.stats)
        margin_min(a.stats, kMarginAlpha, valid ? fabs(alpha - kEpsContrib) / kEpsContrib : 1e300);
}

// ---------------------------------------------------------------------------
// binning

// Binning straight into fixed-capacity tile buckets: the tile counter's old
// value is the entry's slot (any order; k_sort_tiles_* restores depth order).
// Entry = fp32 depth bits (monotone for z > 0; or the input index for the
// composite seam) << 32 | primitive id.  Warp-cooperative: the warp's
// (primitive, tile) pairs are spread over its lanes so that 32 counter
// atomics are in flight per round instead of one serial chain per thread.
// The binning's tile counters sit one per 64 bytes: L2 atomics on
// neighbouring counters of one line serialise (k_bin 235 -> 196 us per C2
// step against dense counters); k_bin_counts compacts them into the dense
// per-tile counts the later kernels read.
#ifndef BIN_COUNT_STRIDE
#define BIN_COUNT_STRIDE 16
#endif
constexpr int kBinCountStride = BIN_COUNT_STRIDE;

__global__ void k_bin_counts(const uint32_t *__restrict__ padded, uint32_t *__restrict__ dense, int64_t n) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) dense[g] = padded[g * kBinCountStride];
}

struct BinArgs {
    const uint2 *binrec;
    const CullRec *cullrec;
    const uint64_t *depth;
    const int32_t *ntiles;
    const int64_t *tile_base;
    const int32_t *tiles_x;
    const int64_t *count;
    uint32_t *tile_count;
    uint64_t *bucket;
    uint32_t cap;
    unsigned int *flags;
    int64_t stride;
    int index_order;
    const int32_t *const *minrank;  // per item clean-tile skip arrays, or null
    const int32_t *keep_min;
};

// SKIP: the clean-tile test of a pruning-level sweep (a separate instantiation:
// the per-pair test costs the probe's binning ~10%)
template <bool SKIP>
__global__ void __launch_bounds__(256) k_bin(BinArgs a) {
    const int s = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t o = (int64_t)s * a.stride + i;
    const int nt = i < a.count[s] ? max(a.ntiles[o], 0) : 0;
    if (__all_sync(0xffffffffu, nt == 0)) return;
    int u0 = 0, u1 = 0, v0 = 0;  // tile range (the last row follows from nt)
    bool cull = false;           // this primitive's pairs pass the ellipse test first
    CullRec cr{};
    uint64_t entry = 0;
    if (nt > 0) {
        const uint2 br = a.binrec[o];  // 8 bytes instead of the 96-byte record
        u0 = (int)(br.x & 0xffffu);
        u1 = (int)((br.x & ~kCullFlag) >> 16);
        v0 = (int)(br.y & 0xffffu);
        if (br.x & kCullFlag) {
            cull = true;
            cr = a.cullrec[o];
        }
        entry = ((uint64_t)list_key32(a.depth[o]) << 32) | (uint32_t)i;
    }
    const int nu = u1 - u0 + 1;
    int incl = nt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    const int excl = incl - nt;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int64_t tb = a.tile_base[s];
    const int txn = a.tiles_x[s];
    // clean tiles of a pruning level take no pairs (k_compositeN skips them)
    const int32_t *mr = SKIP ? a.minrank[s] : nullptr;
    const int32_t kmin = SKIP && mr ? a.keep_min[s] : 0;
    // two rounds of 32 pairs per iteration: both counter atomics are in flight
    // before either result is consumed
    const bool any_cull = __any_sync(0xffffffffu, cull);
    auto resolve = [&](int k, int64_t &g, uint64_t &oent) -> bool {
        // owner lane: the last lane whose first pair index is <= k
        int L = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int e = __shfl_sync(0xffffffffu, excl, L + step);
            if (e <= k) L += step;
        }
        const int j = k - __shfl_sync(0xffffffffu, excl, L);
        const int ou0 = __shfl_sync(0xffffffffu, u0, L), onu = __shfl_sync(0xffffffffu, nu, L);
        const int ov0 = __shfl_sync(0xffffffffu, v0, L);
        oent = __shfl_sync(0xffffffffu, entry, L);
        const int dv = j / onu;
        g = tb + (int64_t)(ov0 + dv) * txn + ou0 + (j - dv * onu);
        // (no early return before the shuffles below: they take the full warp)
        const bool clean = SKIP && mr && k < total && mr[g - tb] >= kmin;
        if (!any_cull) return !clean;  // warp-uniform
        CullRec oc;
        oc.A = __shfl_sync(0xffffffffu, cr.A, L);
        oc.B = __shfl_sync(0xffffffffu, cr.B, L);
        oc.C = __shfl_sync(0xffffffffu, cr.C, L);
        oc.rX = __shfl_sync(0xffffffffu, cr.rX, L);
        oc.rY = __shfl_sync(0xffffffffu, cr.rY, L);
        oc.mx = __shfl_sync(0xffffffffu, cr.mx, L);
        oc.my = __shfl_sync(0xffffffffu, cr.my, L);
        oc.t = __shfl_sync(0xffffffffu, cr.t, L);
        const bool oculled = __shfl_sync(0xffffffffu, cull, L);
        return !clean && (!oculled || cull_keep(oc, j - dv * onu, dv));
    };
    for (int k0 = 0; k0 < total; k0 += 64) {
        const int ka = k0 + lane, kb = k0 + 32 + lane;
        int64_t ga = 0, gb = 0;
        uint64_t ea = 0, eb = 0;
        const bool keepa = resolve(ka, ga, ea);
        const bool keepb = resolve(kb, gb, eb);
        const bool va = ka < total && keepa, vb = kb < total && keepb;
        const uint32_t pa = va ? atomicAdd(a.tile_count + ga * kBinCountStride, 1u) : 0u;
        const uint32_t pb = vb ? atomicAdd(a.tile_count + gb * kBinCountStride, 1u) : 0u;
        if (va) {
            if (pa < a.cap) a.bucket[ga * a.cap + pa] = ea;
            else atomicOr(a.flags, (unsigned)kFlagBucketOverflow);
        }
        if (vb) {
            if (pb < a.cap) a.bucket[gb * a.cap + pb] = eb;
            else atomicOr(a.flags, (unsigned)kFlagBucketOverflow);
        }
    }
}



struct TileScanIn {
    const uint32_t *cnt;
    __device__ int64_t operator()(int, int64_t g) const { return cnt[g]; }
};
struct TileScanOut {
    int64_t *start;
    uint32_t *big_list;  // tiles whose list exceeds the shared-memory sort
    unsigned int *big_n;
    unsigned int *vmax;  // longest list above 256 (bucket capacity adaptation)
    uint32_t cap;
    __device__ void operator()(int, int64_t g, int64_t ex, int64_t v) const {
        start[g] = ex;
        if (v > cap) big_list[atomicAdd(big_n, 1u)] = (uint32_t)g;
        if (v > 256) atomicMax(vmax, (unsigned int)v);
    }
};

struct EmitArgs {
    const Rec *recs;
    const uint2 *binrec;       // cull flag (bit 31 of x)
    const CullRec *cullrec;
    const uint64_t *depth;
    const int32_t *ntiles;
    const int64_t *tile_base;
    const int32_t *tiles_x;
    const int64_t *count;      // primitives per item
    const int64_t *tstart;     // global tile -> first slot
    uint32_t *cursor;          // global tile -> fill cursor
    uint64_t *ids;             // list entries (fp32 depth bits << 32 | id) in tile ranges
    int64_t stride;
    int index_order;           // (informational: the keys themselves decide, see k_bin)
    const int32_t *const *minrank;  // per item clean-tile skip arrays (the pairs k_bin counted), or null
    const int32_t *keep_min;
};

__global__ void __launch_bounds__(256) k_emit(EmitArgs a) {
    const int s = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.count[s]) return;
    const int64_t o = (int64_t)s * a.stride + i;
    if (a.ntiles[o] <= 0) return;
    const Rec &r = a.recs[o];
    const int64_t tb = a.tile_base[s];
    const uint64_t entry = ((uint64_t)list_key32(a.depth[o]) << 32) | (uint32_t)i;
    const int txn = a.tiles_x[s];
    int u0, u1, v0, v1;
    rec_tile_range(r, u0, u1, v0, v1);
    const bool cull = a.binrec && (a.binrec[o].x & kCullFlag);  // the binning's pairs exactly
    CullRec cr{};
    if (cull) cr = a.cullrec[o];
    const int32_t *mr = a.minrank ? a.minrank[s] : nullptr;
    const int32_t kmin = mr ? a.keep_min[s] : 0;
    for (int v = v0; v <= v1; ++v)
        for (int u = u0; u <= u1; ++u) {
            if (cull && !cull_keep(cr, u - u0, v - v0)) continue;
            if (mr && mr[v * txn + u] >= kmin) continue;
            const int64_t g = tb + v * txn + u;
            a.ids[a.tstart[g] + atomicAdd(a.cursor + g, 1u)] = entry;
        }
}

// oversized tiles: gather (key, id) of their ranges for the radix fallback
struct BigArgs {
    const uint32_t *big_list;
    const int64_t *tstart;
    const uint32_t *tcount;
    const int32_t *tile_item;   // global tile -> item
    const uint64_t *depth;      // [nitems][stride]
    uint64_t *ids;
    int64_t stride;
    const int64_t *seg_begin;   // per big tile: offset in the gathered arrays
    uint64_t *keys;
    uint32_t *vals;
};

__global__ void __launch_bounds__(256) k_big_gather(BigArgs a) {
    const int b = blockIdx.y;
    const uint32_t g = a.big_list[b];
    const int64_t n = a.tcount[g], s0 = a.tstart[g], d0 = a.seg_begin[b];
    const int64_t item = a.tile_item[g];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t id = (uint32_t)a.ids[s0 + k];
        a.vals[d0 + k] = id;
        a.keys[d0 + k] = a.depth[item * a.stride + id];
    }
}

__global__ void __launch_bounds__(256) k_big_scatter(BigArgs a, const uint32_t *__restrict__ sorted_vals) {
    const int b = blockIdx.y;
    const uint32_t g = a.big_list[b];
    const int64_t n = a.tcount[g], s0 = a.tstart[g], d0 = a.seg_begin[b];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        a.ids[s0 + k] = sorted_vals[d0 + k];
}

__global__ void __launch_bounds__(256) k_ids_as_keys(const uint32_t *__restrict__ vals, uint64_t *__restrict__ keys,
                                                     int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = vals[i];
}

__global__ void __launch_bounds__(256) k_gather_keys(const uint32_t *__restrict__ vals, const int64_t *__restrict__ seg_begin,
                                                     const uint32_t *__restrict__ big_list, const int32_t *__restrict__ tile_item,
                                                     const uint32_t *__restrict__ tcount, const uint64_t *__restrict__ depth,
                                                     int64_t stride, uint64_t *__restrict__ keys) {
    const int b = blockIdx.y;
    const uint32_t g = big_list[b];
    const int64_t n = tcount[g], d0 = seg_begin[b];
    const int64_t item = tile_item[g];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        keys[d0 + k] = depth[item * stride + vals[d0 + k]];
}

// ---------------------------------------------------------------------------
// compositing

struct CompItem {
    const Rec *recs;         // primitive records of this item
    const uint64_t *depth;   // orderable depth keys of this item
    const double *target;    // (h,w,3) or null
    double *image;           // (h,w,3) or null
    double *trans;           // (h,w) or null
    int64_t *usage;          // [n] or null
    double *sse_tiles;       // per (tile, warp) of this item
    int32_t *term;           // (h,w) terminating primitive or -1 (diagnostic counters only)
    uint32_t *cbits;         // RECORD: contribution bit per (pixel, tile-list entry), or null
    const int64_t *cbase;    // RECORD: first word of each (global) tile's bit block
    int32_t w, h, tiles_x, clip;
};

constexpr double kLog2e = 1.4426950408889634;
// log2(1 / fl(1/255)) rounded to fp32 (threshold offset in the log2 domain)
__device__ __forceinline__ float log2_inv_eps() { return 7.99435343685886f; }

// fp64 constants of the exact path, read as constant-bank operands (no
// per-iteration immediate materialisation)
__constant__ double kCompC[9] = {kExpInvLn2N, kExpNegLn2HiN, kExpNegLn2LoN, kExpC3,     kExpC5,
                                 kExpC4,      kAlphaClamp,   kEpsContrib,   kExpC2};

// exp(x) for the compositing weights, bit-identical to the reference's: the
// table-driven algorithm of glibc 2.39's exp (FMA variant, 128-entry table of
// 2^(i/128) + degree-5 polynomial, same constants and the same fma nesting --
// tools/gen_exp_table.py; tests/test_exp_table.py checks it bit for bit
// against the host libm), which the reference's Cython kernel calls at
// _composite.pyx:57.  The table can be replicated kExpRep times, entry-major,
// with lane l reading copy l % kExpRep, so that the 8 lanes of a 128-bit
// shared-memory phase spread over more bank groups; that paid (x2) for the
// one-pixel kernel, whose limiter was the shared-memory data pipe, but the
// two-pixel union kernel is faster with one copy (less shared memory per CTA):
// 3.24 vs 3.33 ms per C2 step.
#ifndef EXP_REP
#define EXP_REP 1
#endif
constexpr int kExpRep = EXP_REP;

// copy of the exp table for this lane (pass to exp_tab)
template <int REP = kExpRep>
__device__ __forceinline__ const double2 *exp_lane_tab(const double2 *tab) {
    return tab + (threadIdx.x & (REP - 1));
}

template <int REP = kExpRep>
__device__ __forceinline__ void load_exp_table(double2 *tab, int nthreads) {
    const unsigned long long *src = &kExpTable[0][0];
    for (int k = threadIdx.x; k < kExpN * REP; k += nthreads) {
        const int i = k / REP;
        tab[k] = make_double2(__longlong_as_double((long long)src[2 * i]),
                              __longlong_as_double((long long)src[2 * i + 1]));
    }
}

template <int REP = kExpRep>
__device__ __forceinline__ double exp_tab(double x, const double2 *__restrict__ tab) {
    const double shift = 6755399441055744.0;  // 1.5 * 2^52
    const double z = x * kCompC[0];
    double kd = z + shift;
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = kd - shift;
    double r = fma(kd, kCompC[1], x);
    r = fma(kd, kCompC[2], r);
    const double2 t = tab[(ki & (kExpN - 1)) * REP];
    // scale 2^(k/N): add k/N to the table entry's exponent -- only the high word changes
    // ((ki << (52 - kExpBits)) has a zero low word), so one 32-bit add instead of a 64-bit one
    const int sb_hi = __double2hiint(t.y) + (int)((unsigned)ki << (52 - kExpBits - 32));
    const double r2 = r * r;
    const double p1 = fma(r, kCompC[3], kCompC[8]);
    const double p2 = fma(r, kCompC[4], kCompC[5]);
    double tmp = t.x + r;
    tmp = fma(r2, p1, tmp);
    tmp = fma(r2 * r2, p2, tmp);
    const double sc = __hiloint2double(sb_hi, __double2loint(t.y));
    return fma(sc, tmp, sc);
}

constexpr int kCompWarps = kTileThreads / 32;
constexpr int kBatch = 128;             // primitives staged per CTA batch
constexpr int kWarpList = kBatch + 8;   // per-warp compacted list, padded to a multiple of 8

// Per CTA: one staged batch of the tile's depth-ordered list (fp64 fields for
// the exact path, indexed by staged position) and, per warp, the compacted
// sub-list of the batch entries that may touch the warp's 8x4 sub-tile, with
// the fp32 fast-reject fields pair-interleaved for packed f32x2 arithmetic.
struct CompShared {
    double2 m[kBatch];     // mx, my
    double2 hab[kBatch];   // 0.5*a, b
    double2 hcal[kBatch];  // 0.5*c, alpha
    double2 rg[kBatch];    // colour r, g
    double bl[kBatch];     // colour b
    float4 f0[kBatch];     // -(mx-ox), -(my-oy), A, B   (fp32, log2 domain, staged order)
    float2 f1[kBatch];     // C, -L
    uint32_t gid[kBatch];
    int32_t cnt[kBatch];
    uint8_t wmask[kBatch];  // bit w: may touch warp w's 8x4 sub-tile
    int4 bbox[kBatch];      // BBOX mode: clipped bbox x0, x1, y0, y1
    // per warp, entry pairs (a, b): {-mx_a,-mx_b,-my_a,-my_b}, {A_a,A_b,B_a,B_b}, {C_a,C_b,-L_a,-L_b}
    float4 pl[kCompWarps][kWarpList / 2][3];
    uint8_t sidx[kCompWarps][kWarpList];  // compacted position -> staged position
    double2 exptab[kExpN * kExpRep];
};

constexpr int kSortCap = 2048;  // tile lists up to this length are sorted in shared memory
#ifndef COMP_CHUNK
#define COMP_CHUNK 16
#endif
constexpr int kChunk = COMP_CHUNK;  // compacted entries per phase A / phase B round (T refreshed after each)
static_assert(kChunk % 8 == 0 && kChunk <= 32, "chunk");
#ifndef COMP_BRANCHFREE
#define COMP_BRANCHFREE 1
#endif
constexpr bool kLeanComposite = COMP_BRANCHFREE != 0;
#ifndef COMP_MIN_BLOCKS
#define COMP_MIN_BLOCKS 4
#endif
#ifndef COMP_PREFETCH
#define COMP_PREFETCH 1  // 0: none, 1: next batch's records into L1, 2: into L2
#endif

// alpha' = min(al * exp(-e), 0.999) for staged primitive j at (dx, dy):
// exact replay of _composite.pyx:56-60 (0.5*(A + C) == 0.5A + 0.5C exactly)
__device__ __forceinline__ double alpha_at(const CompShared &sh, int j, double pxd, double pyd) {
    const double2 mm = sh.m[j];
    const double2 ab = sh.hab[j];
    const double2 ca = sh.hcal[j];
    const double dx = pxd - mm.x;
    const double dy = pyd - mm.y;
    const double ee = (ab.x * dx * dx + ca.x * dy * dy) + ab.y * dx * dy;
    const double ap = ca.y * exp_tab(-ee, exp_lane_tab(sh.exptab));
    return ap > kCompC[6] ? kCompC[6] : ap;
}

// ---- tile-list sort: ascending (depth key, primitive index) -----------------
// All sorts work on unique 32-bit keys (tile-local depth bucket << position
// bits | list position); see warp_sort_tile and k_sort_tiles_radix.

// ---- per-tile list sort kernels ------------------------------------------------
// One warp per tile, entries e = lane + 32 r held in registers (R per lane);
// the full bitonic network runs with in-lane swaps for strides >= 32 and
// shuffles below -- no shared memory, no barriers.
template <int R, typename K>
__device__ __forceinline__ void warp_reg_bitonic(K (&k)[R]) {
    const int lane = threadIdx.x & 31;
    constexpr int N = 32 * R;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int st = size >> 1; st > 0; st >>= 1) {
            if (st >= 32) {
                const int rs = st >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & rs) continue;
                    const int r2 = r | rs;
                    const bool asc = ((lane + 32 * r) & size) == 0;
                    const K a = k[r], b = k[r2];
                    const bool sw = (a > b) == asc;
                    k[r] = sw ? b : a;
                    k[r2] = sw ? a : b;
                }
            } else {
                const bool lower = (lane & st) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const K p = __shfl_xor_sync(0xffffffffu, k[r], st);
                    const bool asc = ((lane + 32 * r) & size) == 0;
                    k[r] = (lower == asc) ? min(k[r], p) : max(k[r], p);
                }
            }
        }
    }
}

// Tile lists: primitive ids, either in fixed-capacity buckets (list of tile g
// at g * cap) or in scanned ranges (at tstart[g]).
struct TileLists {
    uint64_t *ids;          // entries: fp32 depth bits << 32 | primitive id
    const int64_t *tstart;  // null: buckets
    uint32_t cap;
    __device__ __forceinline__ uint64_t *list(int64_t g) const { return ids + (tstart ? tstart[g] : g * (int64_t)cap); }
    // entries of tile g's list (an overflowed bucket holds only cap of them; such a
    // call is redone through scanned ranges, see bin_and_composite)
    __device__ __forceinline__ int count(const uint32_t *tcount, int64_t g) const {
        const uint32_t n = tcount[g];
        return (int)(tstart ? n : min(n, cap));
    }
};

struct TileSortArgs {
    TileLists tl;
    const uint32_t *tcount;
    const int64_t *tile_base;  // per item
    int nitems;
    const uint64_t *depth;     // [nitems][stride] orderable depth keys
    int64_t stride;
    uint32_t *slow_list;       // tiles needing the block-level exact sort
    unsigned int *slow_n;
    uint32_t *mid_list;        // tiles longer than kWarpSortMax (k_sort_tiles_radix<1024, ...>)
    unsigned int *mid_n;
    int64_t Tt;
};

__device__ __forceinline__ int item_of_tile(const int64_t *__restrict__ tile_base, int nitems, int64_t g) {
    int lo = 0, hi = nitems - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_base[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Sort one tile list (n <= 32 R) in registers on 32-bit keys: each entry's
// fp32 depth bits are re-bucketed to 32 - PB bits over the tile's own range,
// with the entry's list position in the low PB bits (PB = 10, or 11 for lists
// above 1024).  Distinct buckets are strictly depth ordered (fp32 rounding and
// bucketing are monotone), so the bucket sort is the exact order except inside
// runs of equal buckets, where it is list order: those runs (rare, short) are
// re-sorted in place on the exact (64-bit depth key, index) afterwards.
// Only the primitive ids travel on (every consumer of a sorted list reads the
// low word).
template <int R, int PB>
__device__ __forceinline__ void warp_sort_tile(const TileSortArgs &a, int64_t g, int n, uint32_t *sflags) {
    const int lane = threadIdx.x & 31;
    constexpr uint32_t kPMask = (1u << PB) - 1u;
    uint64_t *lst = a.tl.list(g);
    uint32_t key[R];
    uint32_t bmin = 0xffffffffu, bmax = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        const uint32_t b = e < n ? (uint32_t)(lst[e] >> 32) : 0u;
        key[r] = b;
        if (e < n) {
            bmin = min(bmin, b);
            bmax = max(bmax, b);
        }
    }
    bmin = __reduce_min_sync(0xffffffffu, bmin);
    bmax = __reduce_max_sync(0xffffffffu, bmax);
    const uint32_t span = bmax - bmin;
    const int sh = max(0, (32 - __clz((int)span)) - (32 - PB));
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        key[r] = e < n ? (((key[r] - bmin) >> sh) << PB) | (uint32_t)e : 0xffffffffu;
    }
    warp_reg_bitonic<R>(key);
    // adjacent entries in one bucket: their exact order is fixed below
    bool clash = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        const uint32_t nxt_same = __shfl_down_sync(0xffffffffu, key[r], 1);
        const uint32_t nxt_row = __shfl_sync(0xffffffffu, key[r + 1 < R ? r + 1 : r], 0);
        const uint32_t nx = lane < 31 ? nxt_same : nxt_row;
        const bool same = e + 1 < n && (key[r] >> PB) == (nx >> PB);
        clash |= same;
        if (sflags) {
            const unsigned m = __ballot_sync(0xffffffffu, same);
            if (lane == 0) sflags[r] = m;
        }
    }
    // gather the ids in sorted order (in place in key[]), then write them back
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        key[r] = e < n ? (uint32_t)lst[key[r] & kPMask] : 0u;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = lane + 32 * r;
        if (e < n) lst[e] = key[r];
    }
    if (!__any_sync(0xffffffffu, clash)) return;
    if (!sflags) {  // no flag scratch: the exact block sort takes the tile
        if (lane == 0) a.slow_list[atomicAdd(a.slow_n, 1u)] = (uint32_t)g;
        return;
    }
    __syncwarp();  // the written ids and the run flags are visible to the warp
    const uint64_t *depth = a.depth + (int64_t)item_of_tile(a.tile_base, a.nitems, g) * a.stride;
    auto same_next = [&](int e) { return (sflags[e >> 5] >> (e & 31)) & 1u; };
    for (int e = lane; e < n; e += 32) {
        if (!same_next(e) || (e > 0 && same_next(e - 1))) continue;  // not the start of a run
        int end = e + 1;
        while (same_next(end)) ++end;
        // insertion sort of lst[e..end] on (64-bit depth key, index)
        for (int i = e + 1; i <= end; ++i) {
            const uint32_t id = (uint32_t)lst[i];
            const uint64_t k = depth[id];
            int j = i - 1;
            while (j >= e) {
                const uint32_t pj = (uint32_t)lst[j];
                const uint64_t kj = depth[pj];
                if (kj < k || (kj == k && pj < id)) break;
                lst[j + 1] = pj;
                --j;
            }
            lst[j + 1] = id;
        }
    }
}

#ifndef WARP_SORT_MAX
#define WARP_SORT_MAX 512
#endif
constexpr int kWarpSortMax = WARP_SORT_MAX;  // lists up to this length: k_sort_tiles_warp (<= 64 registers)

__global__ void __launch_bounds__(128, 8) k_sort_tiles_warp(TileSortArgs a) {
    __shared__ uint32_t sflags[4][kWarpSortMax / 32];
    const int64_t g = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (g >= a.Tt) return;
    const int n = a.tl.count(a.tcount, g);
    if (n <= 1 || n > kSortCap) return;  // > kSortCap: radix fallback already sorted it
    if (n > kWarpSortMax) {  // the block radix sort (k_sort_tiles_radix) takes it
        if ((threadIdx.x & 31) == 0) a.mid_list[atomicAdd(a.mid_n, 1u)] = (uint32_t)g;
        return;
    }
    uint32_t *fl = sflags[threadIdx.x >> 5];
    if (n <= 32) warp_sort_tile<1, 10>(a, g, n, fl);
    else if (n <= 64) warp_sort_tile<2, 10>(a, g, n, fl);
    else if (n <= 128) warp_sort_tile<4, 10>(a, g, n, fl);
    else if (n <= 256) warp_sort_tile<8, 10>(a, g, n, fl);
    else warp_sort_tile<16, 10>(a, g, n, fl);
}

#ifndef BIG_RADIX
#define BIG_RADIX 128  // threads of the block radix sort for 1025-2048 lists (16 keys each)
#endif

// Block-level sort of long tile lists: 32-bit keys (depth bucket << PB | list
// position, PB = log2 CAP) sorted by a stable block radix sort over the bucket
// bits only (CUB's BlockRadixSort inside this kernel; the positions are already
// ascending), the ids gathered in that order, runs of equal buckets re-sorted
// on the exact (64-bit depth key, index), written back.  MID: the tiles of
// kWarpSortMax < n <= CAP from the mid list (longer ones are forwarded to the
// slow list); otherwise the slow list (n <= kSortCap).
#ifndef SORT_CUB_BITS
#define SORT_CUB_BITS 5
#endif
template <int CAP, int THREADS, bool MID>
__global__ void __launch_bounds__(THREADS) k_sort_tiles_radix(TileSortArgs a) {
    constexpr int kItems = CAP / THREADS;
    constexpr int PB = CAP == 2048 ? 11 : (CAP == 1024 ? 10 : 9);
    static_assert((1 << PB) == CAP, "power-of-two capacity");
    using BlockRadix = cub::BlockRadixSort<uint32_t, THREADS, kItems, cub::NullType, SORT_CUB_BITS>;
    __shared__ typename BlockRadix::TempStorage radix_tmp;
    __shared__ uint32_t skey[CAP];
    __shared__ uint32_t sid[CAP];
    __shared__ uint32_t sred[2][THREADS / 32];
    const unsigned int nlist = MID ? *a.mid_n : *a.slow_n;
    const uint32_t *list = MID ? a.mid_list : a.slow_list;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (unsigned int b = blockIdx.x; b < nlist; b += gridDim.x) {
        __syncthreads();
        const int64_t g = list[b];
        const int n = a.tl.count(a.tcount, g);
        if (MID && n > CAP) {
            if (threadIdx.x == 0) a.slow_list[atomicAdd(a.slow_n, 1u)] = (uint32_t)g;
            continue;
        }
        uint64_t *lst = a.tl.list(g);
        uint32_t bmin = 0xffffffffu, bmax = 0u;
        for (int e = threadIdx.x; e < n; e += THREADS) {
            const uint32_t hb = (uint32_t)(lst[e] >> 32);
            skey[e] = hb;
            bmin = min(bmin, hb);
            bmax = max(bmax, hb);
        }
        bmin = __reduce_min_sync(0xffffffffu, bmin);
        bmax = __reduce_max_sync(0xffffffffu, bmax);
        if (lane == 0) {
            sred[0][w] = bmin;
            sred[1][w] = bmax;
        }
        __syncthreads();
        bmin = 0xffffffffu;
        bmax = 0u;
#pragma unroll
        for (int k = 0; k < THREADS / 32; ++k) {
            bmin = min(bmin, sred[0][k]);
            bmax = max(bmax, sred[1][k]);
        }
        const int sh = max(0, (32 - __clz((int)(bmax - bmin))) - (32 - PB));
        uint32_t keys[kItems];  // blocked: thread t holds entries kItems t ..
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int e = threadIdx.x * kItems + i;
            keys[i] = e < n ? (((skey[e] - bmin) >> sh) << PB) | (uint32_t)e : 0xffffffffu;
        }
        __syncthreads();  // skey reads done before the sort's shared scratch / the write-back below
        BlockRadix(radix_tmp).Sort(keys, PB, 32);
#pragma unroll
        for (int i = 0; i < kItems; ++i) skey[threadIdx.x * kItems + i] = keys[i];
        __syncthreads();
        for (int e = threadIdx.x; e < n; e += THREADS) sid[e] = (uint32_t)lst[skey[e] & (CAP - 1)];
        __syncthreads();
        const uint64_t *depth = a.depth + (int64_t)item_of_tile(a.tile_base, a.nitems, g) * a.stride;
        auto same_next = [&](int e) { return e + 1 < n && (skey[e] >> PB) == (skey[e + 1] >> PB); };
        for (int e = threadIdx.x; e < n; e += THREADS) {
            if (!same_next(e) || (e > 0 && same_next(e - 1))) continue;  // not the start of a run
            int end = e + 1;
            while (same_next(end)) ++end;
            for (int i = e + 1; i <= end; ++i) {  // insertion sort on (64-bit depth key, index)
                const uint32_t id = sid[i];
                const uint64_t kk = depth[id];
                int j = i - 1;
                while (j >= e) {
                    const uint32_t pj = sid[j];
                    const uint64_t kj = depth[pj];
                    if (kj < kk || (kj == kk && pj < id)) break;
                    sid[j + 1] = pj;
                    --j;
                }
                sid[j + 1] = id;
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < n; e += THREADS) lst[e] = sid[e];
    }
}

// Debug capture (airgs_debug_tile_lists): tile g's list length and its
// primitive indices in compositing order (the low 32 bits of each entry).
__global__ void __launch_bounds__(128) k_dump_tiles(TileLists tl, const uint32_t *__restrict__ tcount, int64_t Tt,
                                                    int32_t *__restrict__ counts, int32_t *__restrict__ ids,
                                                    int64_t max_per_tile) {
    const int64_t g = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= Tt) return;
    const int n = tl.count(tcount, g);
    const uint64_t *lst = tl.list(g);
    if (lane == 0) counts[g] = n;
    for (int k = lane; k < n && k < max_per_tile; k += 32) ids[g * max_per_tile + k] = (int32_t)(uint32_t)lst[k];
}

__global__ void __launch_bounds__(256) k_sum_lists(TileLists tl, const uint32_t *__restrict__ tcount, int64_t Tt,
                                                   unsigned long long *out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = g < Tt ? (unsigned long long)tl.count(tcount, g) : 0ull;
    v = warp_reduce_sum(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

// Diagnostic: depth-order margins of the sorted tile lists -- the smallest
// gap (in ulps of the orderable 64-bit depth keys) between adjacent entries
// with distinct depths, and the number of adjacent exact ties (ordered by
// primitive index).  One warp per tile.
__global__ void __launch_bounds__(128) k_depth_gaps(TileSortArgs a, unsigned long long *stats) {
    const int64_t g = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    unsigned long long gmin = ~0ull, ties = 0;
    if (g < a.Tt) {
        const int n = a.tl.count(a.tcount, g);
        const uint64_t *lst = a.tl.list(g);
        const uint64_t *depth = a.depth + (int64_t)item_of_tile(a.tile_base, a.nitems, g) * a.stride;
        for (int k = lane; k + 1 < n; k += 32) {
            const uint64_t z0 = depth[(uint32_t)lst[k]], z1 = depth[(uint32_t)lst[k + 1]];
            if (z1 == z0) ++ties;
            else gmin = min(gmin, (unsigned long long)(z1 - z0));
        }
    }
    ties = warp_reduce_sum(ties);
    margin_min(stats, kMarginDepthGap, gmin == ~0ull ? 1e300 : (double)gmin);
    if (lane == 0 && ties) atomicAdd(stats + kMarginDepthTies, ties);
}

// One CTA = one 16x16 tile, one pixel per thread; warps are 8x4 sub-tiles.
// The tile's primitive list arrives in depth order (k_sort_tiles_*).
// Per batch of kBatch primitives (staged once per CTA), every warp compacts
// the entries whose threshold-ellipse AABB touches its sub-tile into its own
// list, then walks that list in 32-entry chunks: phase A tests the lane's
// pixel against two entries per packed f32x2 instruction sequence (fp32, log2
// domain, proven guard band) and builds a per-lane candidate mask; phase B has
// every lane run its own candidates through the exact fp64 path in depth
// order (two candidates' exp in flight).
// RECORD: write the contribution record (backward passes).  BBOX: test every
// candidate pixel against the primitive's clipped bbox -- needed only for the
// kernel seam, whose caller-supplied bboxes need not contain the primitive's
// contributing pixels (bboxes from the projection always do: outside the
// 3.5-sigma box alpha * g < 1/255).
template <bool USAGE, bool STATS, bool RECORD = false, bool BBOX = false>
__global__ void __launch_bounds__(kTileThreads, COMP_MIN_BLOCKS)
k_composite(const CompItem *__restrict__ items, const int64_t *__restrict__ tile_base, int nitems,
            const TileLists tls, const uint32_t *__restrict__ tcount, unsigned long long *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char comp_smem[];  // > 48 KB: dynamic
    CompShared &sh = *reinterpret_cast<CompShared *>(comp_smem);
    load_exp_table(sh.exptab, kTileThreads);
    // locate item (binary search over tile_base)
    const int64_t g = blockIdx.x;
    int lo = 0, hi = nitems - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_base[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const CompItem *__restrict__ itp = items + lo;
    const int tl = (int)(g - tile_base[lo]);
    const int tiles_x = itp->tiles_x, img_w = itp->w, img_h = itp->h;
    const int tx = tl % tiles_x, ty = tl / tiles_x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int sx = (w & 1) * 8, sy = (w >> 1) * 4;
    const int lx = sx + (lane & 7), ly = sy + (lane >> 3);
    const int ox = tx * kTile, oy = ty * kTile;
    const int px = ox + lx, py = oy + ly;
    const bool inside = px < img_w && py < img_h;
    const float2 px2 = make_float2((float)lx + 0.5f, (float)lx + 0.5f);
    const float2 py2 = make_float2((float)ly + 0.5f, (float)ly + 0.5f);
    const double pxd = (double)px + 0.5, pyd = (double)py + 0.5;
    const Rec *__restrict__ recs = itp->recs;
    const unsigned lt_mask = (1u << lane) - 1u;

    const int n_all = tls.count(tcount, g);
    const uint64_t *__restrict__ glist = tls.list(g);
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
    bool done = !inside;
    int term_id = -1;          // STATS: primitive whose contribution terminated the pixel
    unsigned long long ncon = 0;  // STATS: contributions of this pixel
    double wmar = 1e300, tmar = 1e300;  // STATS: weight / termination test margins (absolute)
    float thr = log2_inv_eps();  // log2(T/EPS); the guard lives in the staged coefficients

    for (int base = 0; base < n_all; base += kBatch) {
        const int nb = min(kBatch, n_all - base);
        // (the previous batch ended with a block-wide __syncthreads_count: every
        // warp is done with the staging arrays this batch overwrites)
        uint32_t gnext = 0xffffffffu;  // next batch's entry of this thread (record prefetch)
        if ((int)threadIdx.x < nb) {
            const int t = threadIdx.x;
            const uint32_t gi = (uint32_t)glist[base + t];
            if (COMP_PREFETCH && base + kBatch + t < n_all) gnext = (uint32_t)glist[base + kBatch + t];
            const Rec r = recs[gi];
            const float mxl = (float)(r.mx - (double)ox), myl = (float)(r.my - (double)oy);
            sh.gid[t] = gi;
            // fast-reject coefficients: log2e * (a/2, b, c/2) with a/2, c/2 scaled by (1 - kappa) so
            // e' = e - kappa*s absorbs the s-proportional guard; the constant guard
            // is folded into L = log2(alpha) + 6e-5 (fp32 fast reject)
            const double kap = 1.0 - 2e-5;
            sh.f0[t] = make_float4(-mxl, -myl, (float)(0.5 * kLog2e * kap * r.ca), (float)(kLog2e * r.cb));
            sh.f1[t] = make_float2((float)(0.5 * kLog2e * kap * r.cc), -(__log2f((float)r.al) + 6e-5f));
            sh.m[t] = make_double2(r.mx, r.my);
            sh.hab[t] = make_double2(0.5 * r.ca, r.cb);
            sh.hcal[t] = make_double2(0.5 * r.cc, r.al);
            sh.rg[t] = make_double2(r.cr, r.cg);
            sh.bl[t] = r.cbl;
            // sub-tile mask: clipped reference bbox AND threshold-ellipse AABB
            // (pixel centres of sub-tile column k span 8k+0.5 .. 8k+7.5, rows 4k+0.5 .. 4k+3.5)
            unsigned xm = 0, ym = 0;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                xm |= (r.x0 < ox + 8 * k + 8 && r.x1 > ox + 8 * k && mxl - r.hx <= 8.0f * k + 7.5f &&
                       mxl + r.hx >= 8.0f * k + 0.5f) ? (1u << k) : 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                ym |= (r.y0 < oy + 4 * k + 4 && r.y1 > oy + 4 * k && myl - r.hy <= 4.0f * k + 3.5f &&
                       myl + r.hy >= 4.0f * k + 0.5f) ? (1u << k) : 0u;
            unsigned mk = 0;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) mk |= (((xm >> (ww & 1)) & (ym >> (ww >> 1))) & 1u) << ww;
            sh.wmask[t] = (uint8_t)mk;
            if (BBOX) sh.bbox[t] = make_int4(r.x0, r.x1, r.y0, r.y1);
            if (USAGE) sh.cnt[t] = 0;
        }
        __syncthreads();
        // the next batch's records travel while this batch is composited (its
        // staging then waits on L1/L2 instead of DRAM latency)
        if (COMP_PREFETCH && gnext != 0xffffffffu) {
            const char *pa = reinterpret_cast<const char *>(recs + gnext);
            if (COMP_PREFETCH == 1) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 95));
            } else {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + 95));
            }
        }
        // compaction: this warp's entries of the batch, in depth order, pair-interleaved
        int ncomp = 0;  // warp-uniform
        if (!__all_sync(0xffffffffu, done)) {
            for (int c0 = 0; c0 < nb; c0 += 32) {
                const int j = c0 + lane;
                const bool hit = j < nb && ((sh.wmask[j] >> w) & 1u);
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (hit) {
                    const int p = ncomp + __popc(bal & lt_mask);
                    const float4 a0 = sh.f0[j];
                    const float2 a1 = sh.f1[j];
                    float *d = reinterpret_cast<float *>(&sh.pl[w][p >> 1][0]) + (p & 1);
                    d[0] = a0.x;
                    d[2] = a0.y;
                    d[4] = a0.z;
                    d[6] = a0.w;
                    d[8] = a1.x;
                    d[10] = a1.y;
                    sh.sidx[w][p] = (uint8_t)j;
                }
                ncomp += __popc(bal);
            }
            // pad to a multiple of 8 with entries that always reject (-L = +inf)
            if (lane < ((8 - (ncomp & 7)) & 7)) {
                const int p = ncomp + lane;
                float *d = reinterpret_cast<float *>(&sh.pl[w][p >> 1][0]) + (p & 1);
                d[0] = 0.0f;
                d[2] = 0.0f;
                d[4] = 0.0f;
                d[6] = 0.0f;
                d[8] = 0.0f;
                d[10] = __int_as_float(0x7f800000);
            }
            __syncwarp();
        }
        for (int c = 0; c < ncomp; c += kChunk) {
            if (__all_sync(0xffffffffu, done)) break;
            // phase A: fp32 candidate bits, two entries per f32x2 op (T as of the
            // chunk start; a larger T only admits more candidates, never fewer)
            unsigned word = 0;
            const float4 *pl = &sh.pl[w][c >> 1][0];
#pragma unroll
            for (int gq = 0; gq < kChunk / 8; ++gq) {
                if (c + 8 * gq >= ncomp) break;  // warp-uniform; the list is padded to 8
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int pr = 4 * gq + q;
                    const float4 p0 = pl[3 * pr], p1 = pl[3 * pr + 1], p2 = pl[3 * pr + 2];
                    const float2 dx = __fadd2_rn(px2, make_float2(p0.x, p0.y));
                    const float2 dy = __fadd2_rn(py2, make_float2(p0.z, p0.w));
                    // e' - L = dx*(A dx + B dy) + (C dy^2 - L)   (log2 units, guard-scaled)
                    const float2 u = __ffma2_rn(make_float2(p1.x, p1.y), dx, __fmul2_rn(make_float2(p1.z, p1.w), dy));
                    const float2 qv = __ffma2_rn(__fmul2_rn(make_float2(p2.x, p2.y), dy), dy, make_float2(p2.z, p2.w));
                    const float2 e = __ffma2_rn(u, dx, qv);
                    // reject iff e' - L > log2(T/EPS) (guard proof: DESIGN.md)
                    word |= (e.x <= thr ? 1u : 0u) << (2 * pr);
                    word |= (e.y <= thr ? 1u : 0u) << (2 * pr + 1);
                }
            }
            if (done) word = 0;
            // phase B: each lane runs its own candidates in depth order (exact fp64)
            const uint8_t *sid = &sh.sidx[w][c];
            while (word) {
                const int j1 = sid[__ffs(word) - 1];
                word &= word - 1;
                const bool two = word != 0;
                const int j2 = two ? sid[__ffs(word) - 1] : j1;
                word &= word - 1;
                double ap1 = alpha_at(sh, j1, pxd, pyd);
                double ap2 = alpha_at(sh, j2, pxd, pyd);
                if (BBOX) {  // outside the caller's bbox the reference never evaluates the pair
                    const int4 b1 = sh.bbox[j1], b2 = sh.bbox[j2];
                    if (px < b1.x || px >= b1.y || py < b1.z || py >= b1.w) ap1 = 0.0;
                    if (px < b2.x || px >= b2.y || py < b2.z || py >= b2.w) ap2 = 0.0;
                }
                if (kLeanComposite && !USAGE && !STATS && !RECORD && !BBOX) {
                    // evaluation variant, branch-free: a non-contributing candidate adds
                    // exactly 0.0 to the (non-negative) colour sums and keeps T by a select
                    const double2 rg1 = sh.rg[j1], rg2 = sh.rg[j2];
                    const double bl1 = sh.bl[j1], bl2 = sh.bl[j2];
                    double wa = ap1 * T;
                    const bool c1 = wa > kCompC[7];
                    wa = c1 ? wa : 0.0;
                    cr += wa * rg1.x;
                    cg += wa * rg1.y;
                    cb += wa * bl1;
                    const double T1 = T * (1.0 - ap1);
                    T = c1 ? T1 : T;
                    double wb = ap2 * T;
                    const bool c2 = two && wb > kCompC[7];
                    wb = c2 ? wb : 0.0;
                    cr += wb * rg2.x;
                    cg += wb * rg2.y;
                    cb += wb * bl2;
                    const double T2 = T * (1.0 - ap2);
                    T = c2 ? T2 : T;
                    continue;
                }
                double wgt = ap1 * T;
                if (STATS) wmar = fmin(wmar, fabs(wgt - kEpsContrib));
                if (wgt > kCompC[7]) {
                    const double2 rg = sh.rg[j1];
                    cr += wgt * rg.x;
                    cg += wgt * rg.y;
                    cb += wgt * sh.bl[j1];
                    T = T * (1.0 - ap1);
                    if (USAGE) atomicAdd(&sh.cnt[j1], 1);
                    if (RECORD) {  // the reference's record=True mask (_composite.pyx:69-71)
                        const int e = base + j1;
                        atomicOr(itp->cbits + itp->cbase[g] + (e >> 5) * kTileThreads + (ly * kTile + lx),
                                 1u << (e & 31));
                    }
                    if (STATS) {
                        ++ncon;
                        if (term_id < 0 && kAlphaClamp * T <= kEpsContrib) term_id = (int)sh.gid[j1];
                        tmar = fmin(tmar, fabs(kAlphaClamp * T - kEpsContrib));
                    }
                }
                if (two) {
                    wgt = ap2 * T;
                    if (STATS) wmar = fmin(wmar, fabs(wgt - kEpsContrib));
                    if (wgt > kCompC[7]) {
                        const double2 rg = sh.rg[j2];
                        cr += wgt * rg.x;
                        cg += wgt * rg.y;
                        cb += wgt * sh.bl[j2];
                        T = T * (1.0 - ap2);
                        if (USAGE) atomicAdd(&sh.cnt[j2], 1);
                        if (RECORD) {
                            const int e = base + j2;
                            atomicOr(itp->cbits + itp->cbase[g] + (e >> 5) * kTileThreads + (ly * kTile + lx),
                                     1u << (e & 31));
                        }
                        if (STATS) {
                            ++ncon;
                            if (term_id < 0 && kAlphaClamp * T <= kEpsContrib) term_id = (int)sh.gid[j2];
                            tmar = fmin(tmar, fabs(kAlphaClamp * T - kEpsContrib));
                        }
                    }
                }
            }
            // once 0.999*T <= EPS no later primitive can pass the weight test
            done = done || kAlphaClamp * T <= kEpsContrib;
            thr = __log2f((float)T) + log2_inv_eps();
        }
        if (USAGE) {  // every warp's shared-memory counts of this batch are final
            __syncthreads();
            if ((int)threadIdx.x < nb && sh.cnt[threadIdx.x] > 0)
                atomicAdd((unsigned long long *)(itp->usage + sh.gid[threadIdx.x]),
                          (unsigned long long)sh.cnt[threadIdx.x]);
        }
        if (__syncthreads_count(!done) == 0) break;
    }

    const CompItem it = *itp;
    const int64_t pix = (int64_t)py * it.w + px;
    double vr = cr, vg = cg, vb = cb;
    if (it.clip) {
        vr = fmin(fmax(vr, 0.0), 1.0);
        vg = fmin(fmax(vg, 0.0), 1.0);
        vb = fmin(fmax(vb, 0.0), 1.0);
    }
    if (inside) {
        if (it.image) {
            it.image[3 * pix] = vr;
            it.image[3 * pix + 1] = vg;
            it.image[3 * pix + 2] = vb;
        }
        if (it.trans) it.trans[pix] = T;
        if (STATS) it.term[pix] = term_id;
    }
    if (STATS) {
        ncon = warp_reduce_sum(ncon);
        if (lane == 0 && ncon) atomicAdd(stats + 2, ncon);
        margin_min(stats, kMarginWeight, wmar / kEpsContrib);
        margin_min(stats, kMarginTerm, tmar / kEpsContrib);
    }
    if (it.target) {
        double se = 0.0;
        if (inside) {
            const double dr = vr - it.target[3 * pix];
            const double dg = vg - it.target[3 * pix + 1];
            const double db = vb - it.target[3 * pix + 2];
            se = (dr * dr + dg * dg) + db * db;
        }
        se = warp_reduce_sum(se);
        if (lane == 0) it.sse_tiles[(int64_t)tl * kCompWarps + w] = se;  // fixed-order reduce later
    }
}

// ---- NP pixels per lane (evaluation and usage passes) -------------------------
// Same per-pixel algorithm as k_composite.  A lane owns NP vertically adjacent
// pixels of one column; a warp owns an SW x 8 sub-tile (NP = 2: 8x8, 4 warps
// per 16x16 tile -- the default; NP = 4: 16x8, 2 warps per tile, measured
// 10% slower: more wasted exps over a 4-way union and 96+ registers).
// Each phase-A broadcast of an entry's fp32 fields serves NP pixel tests and
// the per-warp compaction is amortised over 32*NP pixels; phase B walks the
// union of the lane's NP candidate sets in depth order, one entry per
// iteration, loading its staged fp64 fields once for all NP pixels (the sets
// of adjacent pixels overlap heavily) and sharing dx and fl(fl(a/2 dx) dx);
// the NP exp / blend chains are independent.

#ifndef COMP_PX2
#define COMP_PX2 1
#endif
#ifndef C2_NP
#define C2_NP 2
#endif
#ifndef C2_BATCH
#define C2_BATCH 96
#endif
#ifndef C2_MIN_BLOCKS
#define C2_MIN_BLOCKS (C2_NP == 2 ? 8 : 10)
#endif
#ifndef C2_CHUNK
#define C2_CHUNK 24
#endif
#ifndef C2_STATIC_SMEM
#define C2_STATIC_SMEM 1
#endif
#ifndef C2_SIGNBITS
#define C2_SIGNBITS 1
#endif
#ifndef C2_EXTRA_SMEM
#define C2_EXTRA_SMEM 0
#endif
#ifndef C2_ELLIPSE_CULL
#define C2_ELLIPSE_CULL 0  // measured slower (profiles/r2_composite_experiments.md): off
#endif
#ifndef C2_EXP_REP
#define C2_EXP_REP 1  // 2 and 4 copies measured slower (less L1 left for records)
#endif
// exp table copies of the evaluation kernel: lane l reads copy l % 4, entry-major,
// so a quarter-warp's 128-bit lookups spread over more bank groups
constexpr int kC2ExpRep = C2_EXP_REP;
#ifndef C2_MSB
#define C2_MSB 1  // -0.3% (r2 experiments)
#endif
#ifndef C2_PRED_BLEND
#define C2_PRED_BLEND 1  // predicated blend, no selects: with C2_MSB -1.0% (r2 experiments)
#endif
#ifndef C2_NOCLAMP
#define C2_NOCLAMP 1
#endif
constexpr double kNoClampAlpha = 0.998;
#ifndef C2_PA2
#define C2_PA2 1  // phase A as dy (C dy + B dx) + (A dx dx - L): -1.7% composite (r2 experiments)
#endif

// Lower bound (conservative by 1e-4 of the terms' magnitude + 1e-3, far above
// fp32 rounding) of min Q(dx, dy) = A dx^2 + B dx dy + C dy^2 over the
// rectangle [x0, x1] x [y0, y1] (A, C > 0, positive definite): 0 if the
// rectangle holds the origin, else the smallest of the four edges' minima
// (each a 1-D quadratic minimised at its clamped vertex).
__device__ __forceinline__ float quad_rect_min_lb(float A, float B, float C, float x0, float x1, float y0,
                                                  float y1) {
    if (x0 <= 0.0f && x1 >= 0.0f && y0 <= 0.0f && y1 >= 0.0f) return 0.0f;
    if (!(A > 0.0f && C > 0.0f)) return 0.0f;
    auto edge = [B](float P, float Q, float X, float lo, float hi) {
        // min over t in [lo, hi] of P X^2 + B X t + Q t^2
        const float t = fminf(fmaxf(-B * X / (2.0f * Q), lo), hi);
        const float a = P * X * X, b = B * X * t, c = Q * t * t;
        return (a + b + c) - (1e-4f * (a + fabsf(b) + c) + 1e-3f);
    };
    const float ex = fminf(edge(A, C, x0, y0, y1), edge(A, C, x1, y0, y1));
    const float ey = fminf(edge(C, A, y0, x0, x1), edge(C, A, y1, x0, x1));
    return fminf(ex, ey);
}
constexpr int kC2Chunk = C2_CHUNK;  // compacted entries per phase A / phase B round (24 measured best of 8..32)
static_assert(kC2Chunk % 8 == 0 && kC2Chunk <= 32, "chunk");
constexpr int kC2Batch = C2_BATCH;
constexpr int kC2List = kC2Batch + 8;

template <int NP>
struct CompNGeom {
    static constexpr int kWarps = kTileThreads / (32 * NP);  // warps per tile
    static constexpr int kThreads = 32 * kWarps;
    static constexpr int kSW = 32 * NP / 8;                   // sub-tile width (height 8)
    static constexpr int kLanesPerRow = kSW;                  // lanes across the sub-tile
};

template <int NP, bool USAGE>
struct CompNShared {
    double2 m[kC2Batch];     // mx, my
    double2 hab[kC2Batch];   // 0.5*a, b
    double2 hcal[kC2Batch];  // 0.5*c, alpha
    double2 rg[kC2Batch];    // colour r, g
    double bl[kC2Batch];     // colour b
    float4 f0[kC2Batch];     // -(mx-ox), -(my-oy), A, B
    float2 f1[kC2Batch];     // C, -L
    uint32_t gid[USAGE ? kC2Batch : 1];  // usage pass only
    int32_t cnt[USAGE ? kC2Batch : 1];
    uint8_t wmask[kC2Batch];  // bit w: may touch warp w's sub-tile
    float4 pl[CompNGeom<NP>::kWarps][kC2List / 2][3];
    uint8_t sidx[CompNGeom<NP>::kWarps][kC2List];
    double2 exptab[kExpN * kC2ExpRep];
};

#ifdef C2_COUNT
// experiment builds only (tools/c2_counts.py): work counters of k_compositeN
__device__ unsigned long long g_c2c[10];
#endif

template <bool USAGE, int NP>
__global__ void __launch_bounds__(CompNGeom<NP>::kThreads, C2_MIN_BLOCKS)
k_compositeN(const CompItem *__restrict__ items, const int64_t *__restrict__ tile_base, int nitems,
             const TileLists tls, const uint32_t *__restrict__ tcount) {
    using G = CompNGeom<NP>;
#if C2_STATIC_SMEM
    // static shared memory (< 48 KB): constant shared addresses fold into the
    // load offsets instead of a base-register add per access
    __shared__ CompNShared<NP, USAGE> sh;
#else
    extern __shared__ __align__(16) unsigned char compn_smem[];
    CompNShared<NP, USAGE> &sh = *reinterpret_cast<CompNShared<NP, USAGE> *>(compn_smem);
#endif
    load_exp_table<kC2ExpRep>(sh.exptab, G::kThreads);
    const int64_t g = blockIdx.x;
    int lo = 0, hi = nitems - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_base[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const CompItem *__restrict__ itp = items + lo;
    const int tl = (int)(g - tile_base[lo]);
    const int tiles_x = itp->tiles_x, img_w = itp->w, img_h = itp->h;
    const int tx = tl % tiles_x, ty = tl / tiles_x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int kSubX = kTile / G::kSW;  // sub-tiles across the tile
    const int sx = (w % kSubX) * G::kSW, sy = (w / kSubX) * 8;
    // the lane's NP pixels are vertically adjacent: their candidate sets overlap
    // most, which the phase-B union exploits (rows r, r+4 measured 5% slower at NP = 2)
    const int lx = sx + lane % G::kLanesPerRow, ly0 = sy + NP * (lane / G::kLanesPerRow);
    const int ox = tx * kTile, oy = ty * kTile;
    const int px = ox + lx;
    const float2 px2 = make_float2((float)lx + 0.5f, (float)lx + 0.5f);
    const double pxd = (double)px + 0.5;
    const Rec *__restrict__ recs = itp->recs;
    const unsigned lt_mask = (1u << lane) - 1u;
    const double2 *tab = exp_lane_tab<kC2ExpRep>(sh.exptab);

    const int n_all = tls.count(tcount, g);
    const uint64_t *__restrict__ glist = tls.list(g);
    double T[NP], cr[NP], cg[NP], cb[NP];
    bool done[NP];
    float thr[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        T[k] = 1.0;
        cr[k] = cg[k] = cb[k] = 0.0;
        done[k] = !(px < img_w && oy + ly0 + k < img_h);
        thr[k] = log2_inv_eps();
    }
    if (COMP_PREFETCH && itp->target) {  // the epilogue's target pixels travel into L2 meanwhile
#pragma unroll
        for (int k = 0; k < NP; ++k)
            if (px < img_w && oy + ly0 + k < img_h)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(itp->target + 3 * ((int64_t)(oy + ly0 + k) * img_w + px)));
    }
    auto all_done = [&]() {
        bool d = true;
#pragma unroll
        for (int k = 0; k < NP; ++k) d = d && done[k];
        return d;
    };

    for (int base = 0; base < n_all; base += kC2Batch) {
        const int nb = min(kC2Batch, n_all - base);
        bool hi_alpha = false;
        for (int t = threadIdx.x; t < nb; t += G::kThreads) {
            const uint32_t gi = (uint32_t)glist[base + t];
            if (COMP_PREFETCH && base + kC2Batch + t < n_all) {
                const char *pa = reinterpret_cast<const char *>(recs + (uint32_t)glist[base + kC2Batch + t]);
                asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 95));
            }
            const Rec r = recs[gi];
            const float mxl = (float)(r.mx - (double)ox), myl = (float)(r.my - (double)oy);
            if (USAGE) sh.gid[t] = gi;
            const double kap = 1.0 - 2e-5;
            sh.f0[t] = make_float4(-mxl, -myl, (float)(0.5 * kLog2e * kap * r.ca), (float)(kLog2e * r.cb));
            sh.f1[t] = make_float2((float)(0.5 * kLog2e * kap * r.cc), -(__log2f((float)r.al) + 6e-5f));
            sh.m[t] = make_double2(r.mx, r.my);
            sh.hab[t] = make_double2(0.5 * r.ca, r.cb);
            sh.hcal[t] = make_double2(0.5 * r.cc, r.al);
            sh.rg[t] = make_double2(r.cr, r.cg);
            sh.bl[t] = r.cbl;
            // sub-tiles: columns SW k + 0.5 .. SW k + SW - 0.5, rows 8k + 0.5 .. 8k + 7.5
            unsigned xm = 0, ym = 0;
#pragma unroll
            for (int k = 0; k < kSubX; ++k)
                xm |= (r.x0 < ox + G::kSW * k + G::kSW && r.x1 > ox + G::kSW * k &&
                       mxl - r.hx <= (float)(G::kSW * k + G::kSW) - 0.5f && mxl + r.hx >= (float)(G::kSW * k) + 0.5f)
                          ? (1u << k) : 0u;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                ym |= (r.y0 < oy + 8 * k + 8 && r.y1 > oy + 8 * k && myl - r.hy <= 8.0f * k + 7.5f &&
                       myl + r.hy >= 8.0f * k + 0.5f) ? (1u << k) : 0u;
            unsigned mk = 0;
#pragma unroll
            for (int ww = 0; ww < G::kWarps; ++ww) mk |= (((xm >> (ww % kSubX)) & (ym >> (ww / kSubX))) & 1u) << ww;
#ifdef C2_COUNT
            atomicAdd(&g_c2c[8], (unsigned long long)__popc(mk));
#endif
#if C2_ELLIPSE_CULL
            // exact ellipse test: drop a sub-tile whose pixel-centre rectangle lies
            // wholly outside the phase-A candidate region Q(dx, dy) <= log2(1/EPS) + L
            if (mk && r.hx < 1e29f && r.hy < 1e29f) {
                const float4 f0 = sh.f0[t];
                const float lim = log2_inv_eps() - sh.f1[t].y;
#pragma unroll
                for (int ww = 0; ww < G::kWarps; ++ww) {
                    if (!((mk >> ww) & 1u)) continue;
                    const float x0 = (float)(G::kSW * (ww % kSubX)) + 0.5f + f0.x;
                    const float y0 = 8.0f * (ww / kSubX) + 0.5f + f0.y;
                    if (quad_rect_min_lb(f0.z, f0.w, sh.f1[t].x, x0, x0 + (float)(G::kSW - 1), y0, y0 + 7.0f) > lim)
                        mk &= ~(1u << ww);
                }
            }
#endif
#ifdef C2_COUNT
            atomicAdd(&g_c2c[9], (unsigned long long)__popc(mk));
#endif
            sh.wmask[t] = (uint8_t)mk;
            if (USAGE) sh.cnt[t] = 0;
            hi_alpha |= r.al > kNoClampAlpha;
        }
        const bool batch_clamp = __syncthreads_or(hi_alpha) != 0;
#ifdef C2_COUNT
        if (threadIdx.x == 0) atomicAdd(&g_c2c[5], (unsigned long long)nb);
#endif
        int ncomp = 0;
        if (!__all_sync(0xffffffffu, all_done())) {
            for (int c0 = 0; c0 < nb; c0 += 32) {
                const int j = c0 + lane;
                const bool hit = j < nb && ((sh.wmask[j] >> w) & 1u);
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (hit) {
                    const int p = ncomp + __popc(bal & lt_mask);
                    const float4 a0 = sh.f0[j];
                    const float2 a1 = sh.f1[j];
                    float *d = reinterpret_cast<float *>(&sh.pl[w][p >> 1][0]) + (p & 1);
                    d[0] = a0.x;
                    d[2] = a0.y;
                    d[4] = a0.z;
                    d[6] = a0.w;
                    d[8] = a1.x;
                    d[10] = a1.y;
                    sh.sidx[w][p] = (uint8_t)j;
                }
                ncomp += __popc(bal);
            }
            if (lane < ((8 - (ncomp & 7)) & 7)) {
                const int p = ncomp + lane;
                float *d = reinterpret_cast<float *>(&sh.pl[w][p >> 1][0]) + (p & 1);
                d[0] = 0.0f;
                d[2] = 0.0f;
                d[4] = 0.0f;
                d[6] = 0.0f;
                d[8] = 0.0f;
                d[10] = __int_as_float(0x7f800000);
            }
            __syncwarp();
        }
        for (int c = 0; c < ncomp; c += kC2Chunk) {
            if (__all_sync(0xffffffffu, all_done())) break;
            // phase A: the NP pixels against two entries per f32x2 sequence (dx shared)
            unsigned wd[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) wd[k] = 0;
            const float4 *pl = &sh.pl[w][c >> 1][0];
#if C2_SIGNBITS
            float2 thr2[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) thr2[k] = make_float2(thr[k], thr[k]);
            int ntest = 0;
#endif
#pragma unroll
            for (int gq = 0; gq < kC2Chunk / 8; ++gq) {
                if (c + 8 * gq >= ncomp) break;
#if C2_SIGNBITS
                ntest += 8;
#endif
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int pr = 4 * gq + q;
                    const float4 p0 = pl[3 * pr], p1 = pl[3 * pr + 1], p2 = pl[3 * pr + 2];
                    const float2 A = make_float2(p1.x, p1.y), B = make_float2(p1.z, p1.w);
                    const float2 C = make_float2(p2.x, p2.y), L = make_float2(p2.z, p2.w);
                    const float2 dx = __fadd2_rn(px2, make_float2(p0.x, p0.y));
                    const float2 my = make_float2(p0.z, p0.w);
#if C2_PA2
                    // e' - L = dy (C dy + B dx) + (A dx dx - L): the dx terms once per pair,
                    // 4 packed ops per pixel instead of 5 (same error class as below: every
                    // rounding is relative to terms bounded by 2 (A dx^2 + C dy^2))
                    const float2 Bdx = __fmul2_rn(B, dx);
                    const float2 K = __ffma2_rn(__fmul2_rn(A, dx), dx, L);
#else
                    const float2 Adx = __fmul2_rn(A, dx);
#endif
#pragma unroll
                    for (int k = 0; k < NP; ++k) {
                        const float yk = (float)(ly0 + k) + 0.5f;
                        const float2 dy = __fadd2_rn(make_float2(yk, yk), my);
#if C2_PA2
                        const float2 e = __ffma2_rn(dy, __ffma2_rn(C, dy, Bdx), K);
#else
                        const float2 u = __ffma2_rn(B, dy, Adx);
                        const float2 qv = __ffma2_rn(__fmul2_rn(C, dy), dy, L);
                        const float2 e = __ffma2_rn(u, dx, qv);
#endif
#if C2_SIGNBITS
                        // candidate iff e < thr: the sign bit of fl(e - thr) (exact sign;
                        // e == thr rejects, inside the guard band), appended with one
                        // funnel shift per test (entry order reversed, fixed below)
                        const float2 d = __fadd2_rn(e, make_float2(-thr2[k].x, -thr2[k].y));
                        wd[k] = __funnelshift_l(__float_as_uint(d.x), wd[k], 1);
                        wd[k] = __funnelshift_l(__float_as_uint(d.y), wd[k], 1);
#else
                        wd[k] |= (e.x <= thr[k] ? 1u : 0u) << (2 * pr);
                        wd[k] |= (e.y <= thr[k] ? 1u : 0u) << (2 * pr + 1);
#endif
                    }
                }
            }
#if C2_SIGNBITS
#pragma unroll
            // C2_MSB: keep the funnel-shift order (test i at bit ntest-1-i) and walk it from the
            // most significant bit in phase B (one FLO per entry instead of BREV + FLO)
            for (int k = 0; k < NP; ++k) wd[k] = C2_MSB ? wd[k] : (ntest ? __brev(wd[k]) >> (32 - ntest) : 0u);
#endif
            unsigned wu = 0;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (done[k]) wd[k] = 0;
                wu |= wd[k];
            }
#ifdef C2_COUNT
            {
                unsigned long long cand = 0;
#pragma unroll
                for (int k = 0; k < NP; ++k) cand += __popc(wd[k]);
                const unsigned it = __popc(wu);
                const unsigned long long sc = warp_reduce_sum(cand), si = warp_reduce_sum((unsigned long long)it);
                const unsigned mx = __reduce_max_sync(0xffffffffu, it);
                if (lane == 0) {
                    atomicAdd(&g_c2c[0], sc);
                    atomicAdd(&g_c2c[1], si);
                    atomicAdd(&g_c2c[2], (unsigned long long)mx);
                    atomicAdd(&g_c2c[4], (unsigned long long)min(kC2Chunk, ncomp - c));
                }
            }
#endif
            // phase B: the union of the NP candidate sets in depth order.  The
            // alpha clamp is compiled out for batches whose opacities are all
            // <= kNoClampAlpha: g = exp(-e) <= 1 + 1e-12 (e >= -1e-12: the conic
            // is positive definite, e only rounds), so ap = fl(al g) < 0.999
            // and min(ap, 0.999) = ap exactly.
            const uint8_t *sid = &sh.sidx[w][c];
            auto phase_b = [&](auto clamp_tag) {
                constexpr bool kClamp = decltype(clamp_tag)::value;
#if C2_MSB
                for (; wu;) {
                    const int hb = 31 - __clz(wu);
                    const unsigned bm = 1u << hb;
                    wu ^= bm;
                    const int pos = ntest - 1 - hb;
#define C2_CAND(k) ((wd[k] & bm) != 0u)
#else
                for (; wu; wu &= wu - 1) {
                    const int pos = __ffs(wu) - 1;
#define C2_CAND(k) (((wd[k] >> pos) & 1u) != 0u)
#endif
                    const int j = sid[pos];
                    const double2 mm = sh.m[j], ab = sh.hab[j], ca = sh.hcal[j];
                    const double2 rg = sh.rg[j];
                    const double bl = sh.bl[j];
                    const double dx = pxd - mm.x;
                    const double ex = ab.x * dx * dx;
                    int nc = 0;
#pragma unroll
                    for (int k = 0; k < NP; ++k) {
                        const double dy = ((double)(oy + ly0 + k) + 0.5) - mm.y;
                        const double ee = (ex + ca.x * dy * dy) + ab.y * dx * dy;
                        double ap = ca.y * exp_tab<kC2ExpRep>(-ee, tab);
                        if (kClamp) ap = ap > kCompC[6] ? kCompC[6] : ap;
                        double x = ap * T[k];
                        const bool cp = C2_CAND(k) && x > kCompC[7];
#ifdef C2_COUNT
                        if (cp) atomicAdd(&g_c2c[3], 1ull);
                        if (C2_CAND(k)) {
                            if (kAlphaClamp * T[k] <= kEpsContrib) atomicAdd(&g_c2c[6], 1ull);  // already terminated
                            else if (!cp) atomicAdd(&g_c2c[7], 1ull);  // alive, weight test fails
                        }
#endif
                        if (!USAGE && !C2_PRED_BLEND) {
                            // branch-free: a non-contributing entry adds exact zeros, keeps T
                            x = cp ? x : 0.0;
                            cr[k] += x * rg.x;
                            cg[k] += x * rg.y;
                            cb[k] += x * bl;
                            const double Tn = T[k] * (1.0 - ap);
                            T[k] = cp ? Tn : T[k];
                        } else if (!USAGE) {
                            if (cp) {  // predicated, no selects
                                cr[k] += x * rg.x;
                                cg[k] += x * rg.y;
                                cb[k] += x * bl;
                                T[k] = T[k] * (1.0 - ap);
                            }
                        } else if (cp) {
                            cr[k] += x * rg.x;
                            cg[k] += x * rg.y;
                            cb[k] += x * bl;
                            T[k] = T[k] * (1.0 - ap);
                            ++nc;
                        }
                    }
                    if (USAGE && nc) atomicAdd(&sh.cnt[j], nc);
                }
            };
#undef C2_CAND
            if (C2_NOCLAMP && !batch_clamp)
                phase_b(std::false_type{});
            else
                phase_b(std::true_type{});
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                done[k] = done[k] || kAlphaClamp * T[k] <= kEpsContrib;
                thr[k] = __log2f((float)T[k]) + log2_inv_eps();
            }
        }
        if (USAGE) {
            __syncthreads();
            for (int t = threadIdx.x; t < nb; t += G::kThreads)
                if (sh.cnt[t] > 0)
                    atomicAdd((unsigned long long *)(itp->usage + sh.gid[t]), (unsigned long long)sh.cnt[t]);
        }
        if (__syncthreads_count(!all_done()) == 0) break;
    }

    const CompItem it = *itp;
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int py = oy + ly0 + k;
        double vr = cr[k], vg = cg[k], vb = cb[k];
        const int64_t pix = (int64_t)py * it.w + px;
        if (it.clip) {
            vr = fmin(fmax(vr, 0.0), 1.0);
            vg = fmin(fmax(vg, 0.0), 1.0);
            vb = fmin(fmax(vb, 0.0), 1.0);
        }
        if (px < img_w && py < img_h) {
            if (it.image) {
                it.image[3 * pix] = vr;
                it.image[3 * pix + 1] = vg;
                it.image[3 * pix + 2] = vb;
            }
            if (it.trans) it.trans[pix] = T[k];
            if (it.target) {
                const double dr = vr - it.target[3 * pix];
                const double dg = vg - it.target[3 * pix + 1];
                const double db = vb - it.target[3 * pix + 2];
                sq += (dr * dr + dg * dg) + db * db;
            }
        }
    }
    if (it.target) {
        sq = warp_reduce_sum(sq);
        // the per-tile partial slots (kCompWarps per tile) keep their layout: this kernel's warps, then zeros
        if (lane == 0) {
            it.sse_tiles[(int64_t)tl * kCompWarps + w] = sq;
            for (int k = G::kWarps + w; k < kCompWarps; k += G::kWarps) it.sse_tiles[(int64_t)tl * kCompWarps + k] = 0.0;
        }
    }
}

template <bool USAGE>
static void launch_composite2(int64_t tiles, cudaStream_t st, const CompItem *items, const int64_t *tile_base,
                              int nitems, const TileLists &tl, const uint32_t *tcount) {
    auto *fn = k_compositeN<USAGE, C2_NP>;
    const unsigned grid = (unsigned)tiles;
    if (C2_STATIC_SMEM) {
        // C2_EXTRA_SMEM (experiments): unused dynamic shared memory that caps the
        // CTAs per SM, leaving registers for kernels of another stream
        fn<<<grid, CompNGeom<C2_NP>::kThreads, C2_EXTRA_SMEM, st>>>(items, tile_base, nitems, tl, tcount);
        return;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CompNShared<C2_NP, USAGE>));
    fn<<<grid, CompNGeom<C2_NP>::kThreads, sizeof(CompNShared<C2_NP, USAGE>), st>>>(items, tile_base, nitems, tl,
                                                                                     tcount);
}

// Diagnostic counters: for every (primitive, pixel of its clipped bbox) pair of
// the reference's loop, count it (bbox) and whether the pixel was still live
// there, i.e. the primitive is not behind the pixel's terminating primitive in
// (depth key, index) order.  One thread per primitive; not on the hot path.
__global__ void __launch_bounds__(128)
k_count_pairs(const CompItem *__restrict__ items, const int32_t *__restrict__ ntiles,
              const int64_t *__restrict__ count, int64_t stride, unsigned long long *__restrict__ stats) {
    const int s = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0, nl = 0;
    if (i < count[s] && ntiles[(int64_t)s * stride + i] != 0) {
        const CompItem it = items[s];
        const Rec &r = it.recs[i];
        const uint64_t key = it.depth[i];
        for (int y = r.y0; y < r.y1; ++y)
            for (int x = r.x0; x < r.x1; ++x) {
                const int t = it.term[(int64_t)y * it.w + x];
                ++nb;
                if (t < 0 || key < it.depth[t] || (key == it.depth[t] && i <= t)) ++nl;
            }
    }
    nb = warp_reduce_sum(nb);
    nl = warp_reduce_sum(nl);
    if ((threadIdx.x & 31) == 0 && nb) {
        atomicAdd(stats, nb);
        atomicAdd(stats + 1, nl);
    }
}

// one block per item: fixed-order reduction of that item's tile partials
// (1024 threads, four independent accumulators each: the item's ~45k partials
// are read with enough loads in flight; the order is fixed by the layout)
// Clean tiles of a pruning-level item (airgs_view_item.tile_minrank): the
// binning gave them no pairs, and their pixels equal the target's bit for bit
// (no primitive the level changes reaches them), so their SSE partials are
// exactly 0 -- the same partials compositing their full lists would give.
__global__ void __launch_bounds__(256) k_zero_clean(double *__restrict__ sse_tiles, const int64_t *__restrict__ tile_base,
                                                    const int32_t *const *__restrict__ minrank,
                                                    const int32_t *__restrict__ keep_min) {
    const int s = blockIdx.y;
    const int32_t *mr = minrank[s];
    if (!mr) return;
    const int64_t tl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tl >= tile_base[s + 1] - tile_base[s] || mr[tl] < keep_min[s]) return;
    double *o = sse_tiles + (tile_base[s] + tl) * kCompWarps;
#pragma unroll
    for (int k = 0; k < kCompWarps; ++k) o[k] = 0.0;
}

constexpr int kSseThreads = 1024;
__global__ void __launch_bounds__(kSseThreads)
k_sse_items(const double *__restrict__ sse_tiles, const int64_t *__restrict__ tile_base,
            const uint8_t *__restrict__ has_target, double *__restrict__ out) {
    const int s = blockIdx.x;
    if (!has_target[s]) return;
    const int64_t b = tile_base[s] * kCompWarps, n = (tile_base[s + 1] - tile_base[s]) * kCompWarps;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t k = threadIdx.x;
    for (; k + 3 * kSseThreads < n; k += 4 * kSseThreads) {
        a0 += sse_tiles[b + k];
        a1 += sse_tiles[b + k + kSseThreads];
        a2 += sse_tiles[b + k + 2 * kSseThreads];
        a3 += sse_tiles[b + k + 3 * kSseThreads];
    }
    for (; k < n; k += kSseThreads) a0 += sse_tiles[b + k];
    double acc = warp_reduce_sum((a0 + a1) + (a2 + a3));
    __shared__ double red[kSseThreads / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = warp_reduce_sum(red[threadIdx.x]);
        if (threadIdx.x == 0) out[s] = acc;
    }
}

// generic SSE of two flat arrays (psnr entry point)
__global__ void __launch_bounds__(256)
k_sse_flat_partial(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                   double *__restrict__ part) {
    double acc = 0.0;
    const int64_t per = ceil_div(n, (int64_t)gridDim.x);
    const int64_t lo = per * blockIdx.x, hi = min(n, lo + per);
    for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    acc = warp_reduce_sum(acc);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

__global__ void k_sse_flat_final(const double *__restrict__ part, int nparts, double *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < nparts; ++k) t += part[k];
        *out = t;
    }
}

// build records for the composite seam (inputs already depth ordered)
__global__ void __launch_bounds__(256)
k_seam_records(int64_t k, const double *__restrict__ means2d, const double *__restrict__ conics,
               const double *__restrict__ alphas, const double *__restrict__ colors,
               const int64_t *__restrict__ bboxes, Rec *__restrict__ recs, int32_t *__restrict__ ntiles,
               uint64_t *__restrict__ depth, uint2 *__restrict__ binrec) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    Rec r;
    r.mx = means2d[2 * i];
    r.my = means2d[2 * i + 1];
    r.ca = conics[3 * i];
    r.cb = conics[3 * i + 1];
    r.cc = conics[3 * i + 2];
    r.al = alphas[i];
    r.cr = colors[3 * i];
    r.cg = colors[3 * i + 1];
    r.cbl = colors[3 * i + 2];
    r.x0 = (int32_t)bboxes[4 * i];
    r.x1 = (int32_t)bboxes[4 * i + 1];
    r.y0 = (int32_t)bboxes[4 * i + 2];
    r.y1 = (int32_t)bboxes[4 * i + 3];
    {
        // conic -> covariance diagonal: Sxx = c/det, Syy = a/det (seam inputs are conics)
        const double det = r.ca * r.cc - r.cb * r.cb;
        const double t = log(r.al / kEpsContrib) * 1.0002 + 2e-4;
        const double hx = sqrt(2.0 * fmax(t, 0.0) * (r.cc / det)) * 1.0002 + 1e-3;
        const double hy = sqrt(2.0 * fmax(t, 0.0) * (r.ca / det)) * 1.0002 + 1e-3;
        r.hx = det > 0.0 && isfinite(hx) ? (float)hx * 1.0001f : 1e30f;
        r.hy = det > 0.0 && isfinite(hy) ? (float)hy * 1.0001f : 1e30f;
    }
    recs[i] = r;
    int nt = 0, u0, u1, v0, v1;
    if (r.x1 > r.x0 && r.y1 > r.y0 && rec_tile_range(r, u0, u1, v0, v1)) {
        nt = (u1 - u0 + 1) * (v1 - v0 + 1);
        binrec[i] = make_uint2((uint32_t)u0 | ((uint32_t)u1 << 16), (uint32_t)v0 | ((uint32_t)v1 << 16));
    }
    ntiles[i] = nt > 0 ? nt : (r.x1 > r.x0 && r.y1 > r.y0 ? -1 : 0);
    depth[i] = (uint64_t)i;  // the input order is the depth order
}


__global__ void k_defer_flags(const unsigned int *__restrict__ flags, unsigned int *defer) {
    if (threadIdx.x == 0 && *flags) atomicOr(defer, *flags);
}

__global__ void k_add_i64(int64_t *__restrict__ dst, const int64_t *__restrict__ src, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

// ---------------------------------------------------------------------------
// host orchestration

__global__ void k_tile_item(const int64_t *__restrict__ tile_base, int nitems, int64_t Tt, int32_t *__restrict__ out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Tt) return;
    int lo = 0, hi = nitems - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_base[mid] <= g) lo = mid; else hi = mid - 1;
    }
    out[g] = lo;
}

struct ItemHost {
    int frame, cam;
    int64_t count;  // primitives of its frame
    int w, h, tiles_x, tiles_y;
    const double *target;
    double *image;
    double *trans;
    int64_t *usage;
    int clip;
    const int64_t *frozen = nullptr;  // frozen compositing order positions, or null
    const int32_t *minrank = nullptr; // clean-tile skip (airgs_view_item.tile_minrank), or null
    int32_t keep_min = 0;
};

// Device layout of the per-call descriptors shared by project / emit / composite.
struct Layout {
    int nitems = 0;
    int64_t stride = 0;
    int64_t Tt = 0;                  // total tiles
    std::vector<int64_t> tile_base;  // nitems + 1
    const int64_t *d_tile_base = nullptr;
    const int32_t *d_tiles_x = nullptr;
    const int64_t *d_count = nullptr;
    const int32_t *d_tile_item = nullptr;
    const int32_t *const *d_minrank = nullptr;  // per item: clean-tile skip array or null (null: none at all)
    const int32_t *d_keep_min = nullptr;
};

// Stage B: histogram (already accumulated in tile_count) -> ranges -> emit ->
// oversized-tile fallback sort -> composite -> SSE.
// Fallback binning into scanned ranges: exclusive scan of the (complete) tile
// counts, entries emitted into the ranges, oversized lists presorted by a
// segmented radix sort.  Also adapts the bucket capacity for the next call.
static TileLists scanned_lists(airgs_ctx *ctx, const std::vector<ItemHost> &items, const Layout &L, const Rec *recs,
                               const uint64_t *depth, const int32_t *ntiles, uint32_t *tile_count, int index_order,
                               uint32_t cap, cudaStream_t st, const uint2 *binrec, const CullRec *cullrec) {
    const int nitems = L.nitems;
    int64_t &NL = ctx->launches;
    const int64_t Tt = L.Tt;
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, 8);
    int64_t maxc = 0;
    for (const auto &h : items) maxc = std::max(maxc, h.count);
    // scanned ranges: exclusive scan of the (complete) tile counts, ids emitted
    // into the ranges, oversized tiles presorted by a segmented radix sort
    int64_t *tstart = ctx->scratch_t<int64_t>(kSlotRanges, (size_t)Tt);
    uint32_t *big_list = ctx->scratch_t<uint32_t>(kSlotPairValsAlt, (size_t)Tt);
    unsigned int *big_n = (unsigned int *)(stats + 2);
    unsigned int *vmax = (unsigned int *)(stats + 4);
    int64_t *d_total = stats;
    int64_t *d_Tt = stats + 1;
    AIRGS_CUDA_TRY(cudaMemsetAsync(big_n, 0, sizeof(unsigned int), st));
    AIRGS_CUDA_TRY(cudaMemsetAsync(vmax, 0, sizeof(unsigned int), st));
    h2d_small(ctx, d_Tt, &Tt, sizeof(int64_t), st);
    {
        const int bps = (int)std::max<int64_t>(1, ceil_div(Tt, kScanTile));
        int64_t *blocks = ctx->scratch_t<int64_t>(kSlotScanBlocks, bps);
        seg_scan<int64_t>(TileScanIn{tile_count}, TileScanOut{tstart, big_list, big_n, vmax, (uint32_t)kSortCap},
                          d_Tt, 1, Tt, blocks, d_total, st, &NL);
        check_launch();
    }
    int64_t P = 0;
    unsigned int hbig = 0, hmax = 0;
    AIRGS_CUDA_TRY(cudaMemcpyAsync(&P, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaMemcpyAsync(&hbig, big_n, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaMemcpyAsync(&hmax, vmax, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    {  // adapt the bucket capacity for the next call
        uint32_t c = cap;
        while (c < hmax && c < (uint32_t)kSortCap) c <<= 1;
        ctx->bucket_cap = c;
    }
    uint64_t *ids = ctx->scratch_t<uint64_t>(kSlotPairVals, (size_t)std::max<int64_t>(P, 1));
    uint32_t *cursor = ctx->scratch_t<uint32_t>(kSlotPairKeys, (size_t)Tt);
    AIRGS_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * Tt, st));
    if (P > 0) {
        EmitArgs ea{recs,     binrec,  cullrec, depth,  ntiles,   L.d_tile_base, L.d_tiles_x, L.d_count,
                    tstart,   cursor,  ids,     L.stride, index_order, L.d_minrank, L.d_keep_min};
        k_emit<<<dim3((unsigned)ceil_div(maxc, 256), (unsigned)nitems), 256, 0, st>>>(ea);
        ++NL;
        check_launch();
    }
    if (hbig > 0) {
        // oversized tiles: stable radix sort of each range by index, then by depth key
        std::vector<uint32_t> hlist(hbig);
        AIRGS_CUDA_TRY(cudaMemcpyAsync(hlist.data(), big_list, sizeof(uint32_t) * hbig, cudaMemcpyDeviceToHost, st));
        std::vector<uint32_t> hcnt(hbig);
        for (unsigned b = 0; b < hbig; ++b)
            AIRGS_CUDA_TRY(
                cudaMemcpyAsync(&hcnt[b], tile_count + hlist[b], sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        std::vector<int64_t> seg(2 * hbig);
        int64_t tot = 0, mx = 0;
        for (unsigned b = 0; b < hbig; ++b) {
            seg[b] = tot;
            seg[hbig + b] = hcnt[b];
            tot += hcnt[b];
            mx = std::max<int64_t>(mx, hcnt[b]);
        }
        int32_t *d_tile_item = ctx->scratch_t<int32_t>(kSlotTileItem, (size_t)Tt);
        k_tile_item<<<(unsigned)ceil_div(Tt, 256), 256, 0, st>>>(L.d_tile_base, nitems, Tt, d_tile_item);
        ++NL;
        int64_t *d_seg = ctx->scratch_t<int64_t>(kSlotMisc3, 2 * (size_t)hbig);
        h2d_small(ctx, d_seg, seg.data(), sizeof(int64_t) * 2 * hbig, st);
        uint64_t *k1 = ctx->scratch_t<uint64_t>(kSlotKeys, (size_t)tot);
        uint64_t *k2 = ctx->scratch_t<uint64_t>(kSlotKeysAlt, (size_t)tot);
        uint32_t *v1 = ctx->scratch_t<uint32_t>(kSlotVals, (size_t)tot);
        uint32_t *v2 = ctx->scratch_t<uint32_t>(kSlotValsAlt, (size_t)tot);
        uint32_t *hist = ctx->scratch_t<uint32_t>(kSlotHist, (size_t)hbig * 256 * ceil_div(mx, kSortTile));
        BigArgs ba{big_list, tstart, tile_count, d_tile_item, depth, ids, L.stride, d_seg, k1, v1};
        const dim3 gg((unsigned)std::min<int64_t>(64, ceil_div(mx, 256)), hbig);
        k_big_gather<<<gg, 256, 0, st>>>(ba);
        k_ids_as_keys<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(v1, k1, tot);
        NL += 2;
        bool alt = radix_sort<uint64_t>(k1, v1, k2, v2, d_seg, d_seg + hbig, (int)hbig, mx, 32, hist, st, &NL);
        uint32_t *vs = alt ? v2 : v1;
        uint64_t *ks = alt ? k2 : k1;
        uint64_t *ko = alt ? k1 : k2;
        uint32_t *vo = alt ? v1 : v2;
        k_gather_keys<<<gg, 256, 0, st>>>(vs, d_seg, big_list, d_tile_item, tile_count, depth, L.stride, ks);
        ++NL;
        bool alt2 = radix_sort<uint64_t>(ks, vs, ko, vo, d_seg, d_seg + hbig, (int)hbig, mx, 64, hist, st, &NL);
        k_big_scatter<<<gg, 256, 0, st>>>(ba, alt2 ? vo : vs);
        ++NL;
        check_launch();
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return TileLists{ids, tstart, 0u};
}

// Depth-order every tile list, composite, reduce the per-item SSE.
// Contribution record of a forward pass (the reference's record=True masks,
// _composite.pyx:33-35,69-71) for the backward pass: one bit per (pixel,
// tile-list entry), tile g's block of ceil(n_g / 32) x 256 words at cbase[g].
struct RecordOut {
    TileLists tl{};          // the depth-ordered lists the forward composited
    uint32_t *cbits = nullptr;
    int64_t *cbase = nullptr;
};

struct RecWordsIn {
    const uint32_t *tcount;
    TileLists tl;
    __device__ int64_t operator()(int, int64_t g) const { return (int64_t)((tl.count(tcount, g) + 31) >> 5) * kTileThreads; }
};
struct RecWordsOut {
    int64_t *base;
    __device__ void operator()(int, int64_t g, int64_t ex, int64_t) const { base[g] = ex; }
};

// k_composite instantiations take their CompShared (> 48 KB) as dynamic shared
// memory; the opt-in is a per-function attribute, set before every launch
// (cheap, and correct whichever device is current).
template <bool USAGE, bool STATS, bool RECORD = false, bool BBOX = false>
static void launch_composite(int64_t tiles, cudaStream_t st, const CompItem *items, const int64_t *tile_base,
                             int nitems, const TileLists &tl, const uint32_t *tcount, unsigned long long *stats) {
    auto *fn = k_composite<USAGE, STATS, RECORD, BBOX>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CompShared));
    fn<<<(unsigned)tiles, kTileThreads, sizeof(CompShared), st>>>(items, tile_base, nitems, tl, tcount, stats);
}

static void sort_composite_sse(airgs_ctx *ctx, const std::vector<ItemHost> &items, const Layout &L,
                               const TileLists &tl, const Rec *recs, const uint64_t *depth, const int32_t *ntiles,
                               uint32_t *tile_count, double *sse, cudaStream_t st, RecordOut *rec = nullptr,
                               bool bbox = false) {
    const int nitems = L.nitems;
    int64_t &NL = ctx->launches;
    const int64_t Tt = L.Tt;
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, 8);
    if (Tt > 0) {
        // depth-order every tile list: warp-level register sort, block-level exact sort for the rest
        unsigned int *slow_n = (unsigned int *)(stats + 3);
        uint32_t *slow_list = ctx->scratch_t<uint32_t>(kSlotSlowTiles, 2 * (size_t)Tt);
        AIRGS_CUDA_TRY(cudaMemsetAsync(slow_n, 0, 2 * sizeof(unsigned int), st));
        TileSortArgs ta{tl,          tile_count, L.d_tile_base, nitems,        depth, L.stride,
                        slow_list,   slow_n,     slow_list + Tt, slow_n + 1,   Tt};
        StageScope t_sort(ctx, st, kStageSort);
        k_sort_tiles_warp<<<(unsigned)ceil_div(Tt, 4), 128, 0, st>>>(ta);
        // the long-list block sorts walk device-side tile lists (no host readback)
        k_sort_tiles_radix<1024, 128, true><<<(unsigned)std::min<int64_t>(Tt, 1184), 128, 0, st>>>(ta);
        k_sort_tiles_radix<kSortCap, BIG_RADIX, false><<<(unsigned)std::min<int64_t>(Tt, 1184), BIG_RADIX, 0, st>>>(ta);
        NL += 3;
        check_launch();
        t_sort.end();
        if (ctx->dump.counts) {  // debug capture of the depth-ordered lists (airgs_debug_tile_lists)
            k_dump_tiles<<<(unsigned)ceil_div(Tt, 4), 128, 0, st>>>(tl, tile_count, Tt, ctx->dump.counts,
                                                                   ctx->dump.ids, ctx->dump.max_per_tile);
            ++NL;
            check_launch();
        }
        if (ctx->stats && ctx->d_stats) {  // diagnostic depth-order margins, list entries
            k_depth_gaps<<<(unsigned)ceil_div(Tt, 4), 128, 0, st>>>(ta, ctx->d_stats);
            k_sum_lists<<<(unsigned)ceil_div(Tt, 256), 256, 0, st>>>(tl, tile_count, Tt, ctx->d_stats + kStatTilePairs);
            NL += 2;
            check_launch();
        }
    }
    double *sse_tiles = ctx->scratch_t<double>(kSlotSseTiles, (size_t)Tt * kCompWarps);
    std::vector<CompItem> ci(nitems);
    std::vector<uint8_t> has_t(nitems);
    bool any_usage = false, any_target = false;
    const bool stats_on = ctx->stats && ctx->d_stats;
    int32_t *term = nullptr;
    int64_t maxcount = 0;
    if (stats_on) {
        int64_t px = 0;
        for (const ItemHost &h : items) {
            px += (int64_t)h.w * h.h;
            maxcount = std::max(maxcount, h.count);
        }
        term = ctx->scratch_t<int32_t>(kSlotTerm, (size_t)std::max<int64_t>(px, 1));
    }
    int64_t term_off = 0;
    for (int s = 0; s < nitems; ++s) {
        const ItemHost &h = items[s];
        CompItem &c = ci[s];
        c.recs = recs + (int64_t)s * L.stride;
        c.depth = depth + (int64_t)s * L.stride;
        c.target = h.target;
        c.image = h.image;
        c.trans = h.trans;
        c.usage = h.usage;
        c.sse_tiles = sse_tiles + L.tile_base[s] * kCompWarps;
        c.term = term ? term + term_off : nullptr;
        term_off += (int64_t)h.w * h.h;
        c.w = h.w;
        c.h = h.h;
        c.tiles_x = h.tiles_x;
        c.clip = h.clip;
        any_usage |= h.usage != nullptr;
        any_target |= h.target != nullptr;
        has_t[s] = h.target != nullptr;
    }
    if (rec && Tt > 0) {  // record layout: exclusive scan of the per-tile bit-block sizes
        int64_t *cbase = ctx->scratch_t<int64_t>(kSlotRecBase, (size_t)Tt + 1);
        int64_t *d_Tt = stats + 5, *d_total = stats + 6;
        h2d_small(ctx, d_Tt, &Tt, sizeof(int64_t), st);
        int64_t *blocks = ctx->scratch_t<int64_t>(kSlotScanBlocks, (size_t)std::max<int64_t>(1, ceil_div(Tt, kScanTile)));
        seg_scan<int64_t>(RecWordsIn{tile_count, tl}, RecWordsOut{cbase}, d_Tt, 1, Tt, blocks, d_total, st, &NL);
        check_launch();
        int64_t words = 0;
        AIRGS_CUDA_TRY(cudaMemcpyAsync(&words, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        uint32_t *cbits = ctx->scratch_t<uint32_t>(kSlotRecBits, (size_t)std::max<int64_t>(words, 1));
        AIRGS_CUDA_TRY(cudaMemsetAsync(cbits, 0, sizeof(uint32_t) * std::max<int64_t>(words, 1), st));
        for (CompItem &c : ci) {
            c.cbits = cbits;
            c.cbase = cbase;
        }
        rec->tl = tl;
        rec->cbits = cbits;
        rec->cbase = cbase;
    }
    CompItem *d_ci = (CompItem *)ctx->scratch(kSlotMisc1, sizeof(CompItem) * nitems);
    uint8_t *d_has = (uint8_t *)ctx->scratch(kSlotMisc2, nitems);
    h2d_small(ctx, d_ci, ci.data(), sizeof(CompItem) * nitems, st);
    h2d_small(ctx, d_has, has_t.data(), nitems, st);
    StageScope t_comp(ctx, st, kStageComposite, Tt > 0);
    if (Tt > 0) {
        unsigned long long *cs = ctx->d_stats;
        if (bbox) {  // the kernel seam (caller-supplied bboxes)
            if (rec) {
                if (any_usage)
                    launch_composite<true, false, true, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
                else
                    launch_composite<false, false, true, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
            } else if (any_usage) {
                launch_composite<true, false, false, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
            } else {
                launch_composite<false, false, false, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
            }
        } else if (rec) {
            if (any_usage)
                launch_composite<true, false, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
            else
                launch_composite<false, false, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
        } else if (stats_on) {
            if (any_usage)
                launch_composite<true, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
            else
                launch_composite<false, true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
        } else if (COMP_PX2) {
            if (any_usage)
                launch_composite2<true>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count);
            else
                launch_composite2<false>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count);
        } else if (any_usage) {
            launch_composite<true, false>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
        } else {
            launch_composite<false, false>(Tt, st, d_ci, L.d_tile_base, nitems, tl, tile_count, cs);
        }
        ++NL;
        check_launch();
    }
    if (stats_on && maxcount > 0) {
        // bbox / live pair counts of the reference's Gaussian-major loop
        k_count_pairs<<<dim3((unsigned)ceil_div(maxcount, 128), nitems), 128, 0, st>>>(d_ci, ntiles, L.d_count,
                                                                                       L.stride, ctx->d_stats);
        ++NL;
        check_launch();
    }
    t_comp.end();
    if (sse && any_target) {
        StageScope t_sse(ctx, st, kStageSse);
        if (L.d_minrank) {  // clean tiles of a pruning level: their pixels equal the target, SSE exactly 0
            int64_t maxt = 0;
            for (int s = 0; s < nitems; ++s) maxt = std::max(maxt, L.tile_base[s + 1] - L.tile_base[s]);
            k_zero_clean<<<dim3((unsigned)ceil_div(maxt, 256), (unsigned)nitems), 256, 0, st>>>(
                sse_tiles, L.d_tile_base, L.d_minrank, L.d_keep_min);
            ++NL;
        }
        k_sse_items<<<nitems, kSseThreads, 0, st>>>(sse_tiles, L.d_tile_base, d_has, sse);
        ++NL;
        check_launch();
        t_sse.end();
    }
    // small uploads travel as kernel parameters: nothing host-side must outlive the launches
}

static void bin_and_composite(airgs_ctx *ctx, const std::vector<ItemHost> &items, const Layout &L,
                              const Rec *recs, const uint64_t *depth, const int32_t *ntiles, uint32_t *tile_count,
                              int index_order, double *sse, cudaStream_t st, unsigned int *flags,
                              const uint2 *binrec, const CullRec *cullrec, RecordOut *rec = nullptr) {
    const int nitems = L.nitems;
    int64_t &NL = ctx->launches;
    const int64_t Tt = L.Tt;
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, 8);
    int64_t maxc = 0;
    for (const auto &h : items) maxc = std::max(maxc, h.count);
    // binning straight into fixed-capacity tile buckets (capacity adapted after an overflow)
    const uint32_t cap = ctx->bucket_cap;
    uint64_t *bucket = ctx->scratch_t<uint64_t>(kSlotPairKeysAlt, (size_t)std::max<int64_t>(Tt, 1) * cap);
    if (maxc > 0 && Tt > 0) {
        uint32_t *pad = tile_count;
        if (kBinCountStride > 1) {
            pad = ctx->scratch_t<uint32_t>(kSlotBinCount, (size_t)Tt * kBinCountStride);
            AIRGS_CUDA_TRY(cudaMemsetAsync(pad, 0, sizeof(uint32_t) * (size_t)Tt * kBinCountStride, st));
        }
        BinArgs ba{binrec, cullrec, depth, ntiles, L.d_tile_base, L.d_tiles_x, L.d_count, pad, bucket, cap, flags,
                   L.stride, index_order, L.d_minrank, L.d_keep_min};
        StageScope t_bin(ctx, st, kStageBin);
        const dim3 bgrid((unsigned)ceil_div(maxc, 256), (unsigned)nitems);
        if (L.d_minrank)
            k_bin<true><<<bgrid, 256, 0, st>>>(ba);
        else
            k_bin<false><<<bgrid, 256, 0, st>>>(ba);
        ++NL;
        if (kBinCountStride > 1) {
            k_bin_counts<<<(unsigned)ceil_div(Tt, 256), 256, 0, st>>>(pad, tile_count, Tt);
            ++NL;
        }
        check_launch();
        t_bin.end();
    }
    // usage counts are ADDED to the caller's arrays (airgs_b200.h): accumulate
    // this call's counts in zeroed scratch first, so that a redone call cannot
    // count twice, and add them once at the end
    std::vector<ItemHost> work(items);
    std::vector<std::pair<int64_t *, int64_t *>> usage_map;  // (caller array, scratch)
    {
        int64_t total = 0;
        std::vector<std::pair<int64_t *, int64_t>> uniq;
        for (const ItemHost &h : items)
            if (h.usage && std::find_if(uniq.begin(), uniq.end(), [&](const std::pair<int64_t *, int64_t> &u) {
                               return u.first == h.usage;
                           }) == uniq.end()) {
                uniq.push_back({h.usage, h.count});
                total += h.count;
            }
        if (total > 0) {
            int64_t *scratch = ctx->scratch_t<int64_t>(kSlotUsage, (size_t)total);
            AIRGS_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(int64_t) * total, st));
            int64_t off = 0;
            for (const auto &u : uniq) {
                usage_map.push_back({u.first, scratch + off});
                off += u.second;
            }
            for (ItemHost &h : work)
                if (h.usage)
                    for (const auto &m : usage_map)
                        if (m.first == h.usage) h.usage = m.second;
        }
    }
    TileLists tl{bucket, nullptr, cap};
    sort_composite_sse(ctx, work, L, tl, recs, depth, ntiles, tile_count, sse, st, rec, index_order != 0);
    if (ctx->defer) {  // deferred checking: fold the flags on the device, no synchronisation
        k_defer_flags<<<1, 32, 0, st>>>(flags, ctx->d_defer);
        ++NL;
        check_launch();
        for (const auto &m : usage_map) {
            int64_t n = 0;
            for (const ItemHost &h : items)
                if (h.usage == m.first) n = h.count;
            if (n > 0) {
                k_add_i64<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(m.first, m.second, n);
                ++NL;
            }
        }
        return;
    }
    // one host synchronisation per render: parameter validity and bucket overflow
    unsigned int hflags = 0;
    AIRGS_CUDA_TRY(cudaMemcpyAsync(&hflags, flags, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    if (hflags & kFlagInvalidParam)
        throw ApiFailure(AIRGS_E_VALIDATION, "frame contains invalid primitive parameters");
    if (hflags & kFlagBucketOverflow) {
        // some tile outgrew its bucket: redo this call through scanned ranges
        // (images and SSE are overwritten, the usage scratch is reset)
        for (size_t k = 0; k < usage_map.size(); ++k) {
            int64_t n = 0;
            for (const ItemHost &h : items)
                if (h.usage == usage_map[k].first) n = h.count;
            AIRGS_CUDA_TRY(cudaMemsetAsync(usage_map[k].second, 0, sizeof(int64_t) * n, st));
        }
        const TileLists tl2 =
            scanned_lists(ctx, items, L, recs, depth, ntiles, tile_count, index_order, cap, st, binrec, cullrec);
        sort_composite_sse(ctx, work, L, tl2, recs, depth, ntiles, tile_count, sse, st, rec, index_order != 0);
    }
    for (const auto &m : usage_map) {
        int64_t n = 0;
        for (const ItemHost &h : items)
            if (h.usage == m.first) n = h.count;
        if (n > 0) {
            k_add_i64<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(m.first, m.second, n);
            ++NL;
            check_launch();
        }
    }
}

// Upload per-item layout arrays (tile bases, tiles_x, counts, tile -> item map).
static void upload_layout(airgs_ctx *ctx, const std::vector<ItemHost> &items, Layout &L, cudaStream_t st) {
    const int nitems = (int)items.size();
    L.nitems = nitems;
    L.tile_base.assign(nitems + 1, 0);
    for (int s = 0; s < nitems; ++s) L.tile_base[s + 1] = L.tile_base[s] + (int64_t)items[s].tiles_x * items[s].tiles_y;
    L.Tt = L.tile_base[nitems];
    size_t off = 0;
    auto align = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t o_tb = off; off = align(off + sizeof(int64_t) * (nitems + 1));
    const size_t o_tx = off; off = align(off + sizeof(int32_t) * nitems);
    const size_t o_cnt = off; off = align(off + sizeof(int64_t) * nitems);
    bool any_skip = false;
    for (const ItemHost &h : items) any_skip |= h.minrank != nullptr;
    const size_t o_mr = off; off = align(off + (any_skip ? sizeof(void *) * nitems : 0));
    const size_t o_km = off; off = align(off + (any_skip ? sizeof(int32_t) * nitems : 0));
    std::vector<char> hbuf(off);
    memcpy(hbuf.data() + o_tb, L.tile_base.data(), sizeof(int64_t) * (nitems + 1));
    for (int s = 0; s < nitems; ++s) {
        const int32_t tx = items[s].tiles_x;
        memcpy(hbuf.data() + o_tx + sizeof(int32_t) * s, &tx, sizeof(int32_t));
        memcpy(hbuf.data() + o_cnt + sizeof(int64_t) * s, &items[s].count, sizeof(int64_t));
        if (any_skip) {
            memcpy(hbuf.data() + o_mr + sizeof(void *) * s, &items[s].minrank, sizeof(void *));
            memcpy(hbuf.data() + o_km + sizeof(int32_t) * s, &items[s].keep_min, sizeof(int32_t));
        }
    }
    char *d = (char *)ctx->scratch(kSlotMisc0, off);
    h2d_small(ctx, d, hbuf.data(), off, st);
    L.d_tile_base = (const int64_t *)(d + o_tb);
    L.d_tiles_x = (const int32_t *)(d + o_tx);
    L.d_count = (const int64_t *)(d + o_cnt);
    L.d_tile_item = nullptr;  // built on device when the oversized-tile path needs it
    L.d_minrank = any_skip ? (const int32_t *const *)(d + o_mr) : nullptr;
    L.d_keep_min = any_skip ? (const int32_t *)(d + o_km) : nullptr;
}


// What a backward pass needs from its (recomputed) forward pass.
struct BwdState {
    RecordOut rec;
    const Rec *recs = nullptr;
    double *t_final = nullptr;  // set by the caller: forward writes (h, w)
    int64_t Tt = 0;
    const int64_t *tile_base = nullptr;
    uint32_t *tile_count = nullptr;
};

static void render_impl(airgs_ctx *ctx, const airgs_frame *frames, int nframes, const airgs_camera *cams,
                        int ncams, const airgs_view_item *items, int nitems, double *sse, cudaStream_t st,
                        BwdState *bwd = nullptr) {
    if (nitems <= 0) return;
    if (nframes <= 0 || ncams <= 0) throw ApiFailure(AIRGS_E_STRUCTURAL, "no frames or cameras");
    std::vector<ItemHost> ih(nitems);
    std::vector<std::vector<int32_t>> per_frame(nframes);
    int64_t stride = 0;
    for (int s = 0; s < nitems; ++s) {
        const airgs_view_item &v = items[s];
        if (v.frame < 0 || v.frame >= nframes || v.camera < 0 || v.camera >= ncams)
            throw ApiFailure(AIRGS_E_STRUCTURAL, "view item references a missing frame or camera");
        const airgs_frame &f = frames[v.frame];
        if (f.count <= 0) throw ApiFailure(AIRGS_E_STRUCTURAL, "cannot render an empty frame");
        if (f.width != 17 && f.width != 26)
            throw ApiFailure(AIRGS_E_STRUCTURAL, "no sh degree yields parameter width " + std::to_string(f.width));
        // (list keys hold frozen positions below 2^30)
        if (f.count >= (1LL << 30)) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");
        const airgs_camera &c = cams[v.camera];
        if (c.width < 1 || c.height < 1) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad camera resolution");
        if (c.width > (65535 * kTile) || c.height > (65535 * kTile))
            throw ApiFailure(AIRGS_E_CAPACITY, "camera resolution beyond the tile index range");
        ItemHost &h = ih[s];
        h.frame = v.frame;
        h.cam = v.camera;
        h.count = f.count;
        h.w = c.width;
        h.h = c.height;
        h.tiles_x = (c.width + kTile - 1) / kTile;
        h.tiles_y = (c.height + kTile - 1) / kTile;
        h.target = v.target;
        h.image = v.image;
        h.trans = bwd ? bwd->t_final : nullptr;
        h.usage = v.usage;
        h.frozen = v.frozen_pos;
        h.minrank = v.tile_minrank;
        h.keep_min = v.tile_keep_min;
        if (h.minrank && (!h.target || h.image || h.usage || bwd))
            throw ApiFailure(AIRGS_E_STRUCTURAL, "tile_minrank needs an SSE-only item (target set, no image or usage)");
        h.clip = bwd ? 0 : 1;  // the forward of render_forward returns the unclipped image
        per_frame[v.frame].push_back(s);
        stride = std::max(stride, f.count);
    }
    int64_t &NL = ctx->launches;
    Layout L;
    L.stride = stride;
    upload_layout(ctx, ih, L, st);
    // descriptors -> device (one packed upload)
    std::vector<int32_t> fptr(nframes + 1), fitems, icam(nitems);
    fptr[0] = 0;
    for (int f = 0; f < nframes; ++f) {
        for (int32_t s : per_frame[f]) fitems.push_back(s);
        fptr[f + 1] = (int32_t)fitems.size();
    }
    for (int s = 0; s < nitems; ++s) icam[s] = ih[s].cam;
    size_t off = 0;
    auto align = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t o_frames = off; off = align(off + sizeof(airgs_frame) * nframes);
    const size_t o_cams = off; off = align(off + sizeof(airgs_camera) * ncams);
    const size_t o_fptr = off; off = align(off + sizeof(int32_t) * (nframes + 1));
    const size_t o_fitems = off; off = align(off + sizeof(int32_t) * nitems);
    const size_t o_icam = off; off = align(off + sizeof(int32_t) * nitems);
    bool any_frozen = false;
    for (int s = 0; s < nitems; ++s) any_frozen |= ih[s].frozen != nullptr;
    const size_t o_frz = off; off = align(off + (any_frozen ? sizeof(const int64_t *) * nitems : 0));
    char *hs = (char *)ctx->staging(off);
    memcpy(hs + o_frames, frames, sizeof(airgs_frame) * nframes);
    memcpy(hs + o_cams, cams, sizeof(airgs_camera) * ncams);
    memcpy(hs + o_fptr, fptr.data(), sizeof(int32_t) * (nframes + 1));
    memcpy(hs + o_fitems, fitems.data(), sizeof(int32_t) * nitems);
    memcpy(hs + o_icam, icam.data(), sizeof(int32_t) * nitems);
    if (any_frozen)
        for (int s = 0; s < nitems; ++s) memcpy(hs + o_frz + sizeof(const int64_t *) * s, &ih[s].frozen, sizeof(void *));
    char *dd = (char *)ctx->scratch(kSlotDesc, off);
    h2d_small(ctx, dd, hs, off, st);

    unsigned int *flags = ctx->scratch_t<unsigned int>(kSlotFlags, 4);
    AIRGS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(unsigned int), st));
    const size_t per = (size_t)nitems * stride;
    Rec *recs = ctx->scratch_t<Rec>(kSlotRecs, per);
    uint64_t *depth = ctx->scratch_t<uint64_t>(kSlotDepth, per);
    int32_t *ntiles = ctx->scratch_t<int32_t>(kSlotNtiles, per);
    uint2 *binrec = ctx->scratch_t<uint2>(kSlotBinRec, per);
    CullRec *cullrec = TILE_CULL ? ctx->scratch_t<CullRec>(kSlotCullRec, per) : nullptr;
    uint32_t *tile_count = ctx->scratch_t<uint32_t>(kSlotTileCount, (size_t)L.Tt);
    AIRGS_CUDA_TRY(cudaMemsetAsync(tile_count, 0, sizeof(uint32_t) * L.Tt, st));

    ProjArgs pa;
    pa.frames = (const airgs_frame *)(dd + o_frames);
    pa.cams = (const airgs_camera *)(dd + o_cams);
    pa.frame_item_ptr = (const int32_t *)(dd + o_fptr);
    pa.frame_items = (const int32_t *)(dd + o_fitems);
    pa.item_cam = (const int32_t *)(dd + o_icam);
    pa.item_frozen = any_frozen ? (const int64_t *const *)(dd + o_frz) : nullptr;
    pa.tile_base = L.d_tile_base;
    pa.tiles_x = L.d_tiles_x;
    pa.recs = recs;
    pa.depth = depth;
    pa.ntiles = ntiles;
    pa.binrec = binrec;
    pa.cullrec = cullrec;
    pa.flags = flags;
    pa.stride = stride;
    pa.stats = (ctx->stats && ctx->d_stats) ? ctx->d_stats : nullptr;
    StageScope t_proj(ctx, st, kStageProject);
    {
        dim3 grid((unsigned)ceil_div(stride, kProjThreads), (unsigned)nframes);
        bool all17 = true;
        for (int f = 0; f < nframes; ++f) all17 &= frames[f].width == 17;
        if (all17)
            k_project<17><<<grid, kProjThreads, 0, st>>>(pa);
        else
            k_project<26><<<grid, kProjThreads, 0, st>>>(pa);
        ++NL;
        check_launch();
    }
    t_proj.end();
    bin_and_composite(ctx, ih, L, recs, depth, ntiles, tile_count, 0, sse, st, flags, binrec, cullrec,
                      bwd ? &bwd->rec : nullptr);
    if (bwd) {
        bwd->recs = recs;
        bwd->Tt = L.Tt;
        bwd->tile_base = L.d_tile_base;
        bwd->tile_count = tile_count;
    }
}

// ---------------------------------------------------------------------------
// backward (training): _composite.backward
// (ss/_composite.pyx:77-152) and the projection chain rule of render_backward
// (ss/rasterizer.py:270-369).

constexpr int kBwdBatch = 128;
struct BwdShared {
    double f[9][kBwdBatch];    // mx, my, a, b, c, al, cr, cg, cb of the staged entries
    uint32_t gid[kBwdBatch];
    double2 exptab[kExpN * kExpRep];
};


// One CTA per tile, one pixel per thread: the pixel's recorded contributors in
// reverse depth order with the reference's per-pixel recurrences (t_before =
// T / (1 - ap), the running colour accumulator, d_ap with the clamp rule);
// each warp sums an entry's 9 per-contribution terms over its contributing
// pixels and sends them to the per-primitive totals G[id][9] as native fp64
// L2 reductions (RED.ADD.F64; shared-memory fp64 atomicAdd is a CAS loop on
// sm_100 -- accumulating the terms there made the training step 37% slower).
// The cross-pixel summation order differs from the reference's row-major
// loop; the per-pixel terms do not.
__global__ void __launch_bounds__(kTileThreads) k_composite_bwd(const Rec *__restrict__ recs, const TileLists tls,
                                                               const uint32_t *__restrict__ tcount,
                                                               const uint32_t *__restrict__ cbits,
                                                               const int64_t *__restrict__ cbase, int tiles_x, int w,
                                                               int h, const double *__restrict__ t_final,
                                                               const double *__restrict__ d_image,
                                                               double *__restrict__ G) {
    __shared__ BwdShared sh;
    load_exp_table(sh.exptab, kTileThreads);
    const int64_t g = blockIdx.x;
    const int tx = (int)(g % tiles_x), ty = (int)(g / tiles_x);
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4, lane = threadIdx.x & 31;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < w && py < h;
    const int64_t pix = (int64_t)py * w + px;
    double T = inside ? t_final[pix] : 1.0;
    double dc0 = 0.0, dc1 = 0.0, dc2 = 0.0;
    if (inside) {
        dc0 = d_image[3 * pix];
        dc1 = d_image[3 * pix + 1];
        dc2 = d_image[3 * pix + 2];
    }
    double ac0 = 0.0, ac1 = 0.0, ac2 = 0.0;
    const double pxd = (double)px + 0.5, pyd = (double)py + 0.5;
    const int n = tls.count(tcount, g);
    const uint64_t *lst = tls.list(g);
    const uint32_t *bits = cbits + cbase[g] + threadIdx.x;
    for (int hi = n; hi > 0; hi -= kBwdBatch) {
        const int lo = max(0, hi - kBwdBatch), nb = hi - lo;
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            const int t = threadIdx.x;
            const uint32_t id = (uint32_t)lst[lo + t];
            const Rec &r = recs[id];
            sh.gid[t] = id;
            sh.f[0][t] = r.mx;
            sh.f[1][t] = r.my;
            sh.f[2][t] = r.ca;
            sh.f[3][t] = r.cb;
            sh.f[4][t] = r.cc;
            sh.f[5][t] = r.al;
            sh.f[6][t] = r.cr;
            sh.f[7][t] = r.cg;
            sh.f[8][t] = r.cbl;
        }
        __syncthreads();
        // entry-synchronous per warp: the union of the warp's contributors of
        // each bit word, in reverse depth order (each pixel still sees its own
        // contributors in its own reverse order); an entry's 9 terms are summed
        // over the warp's contributing lanes before they go to L2, so an entry
        // costs 9 reductions per warp instead of 9 per contributing pixel
        for (int wd = (hi - 1) >> 5; wd >= (lo >> 5); --wd) {
            uint32_t m = inside ? bits[(int64_t)wd * kTileThreads] : 0u;
            const int e0 = wd << 5;
            if (e0 < lo) m &= ~0u << (lo - e0);
            if (e0 + 32 > hi) m &= (hi - e0) >= 32 ? ~0u : ((1u << (hi - e0)) - 1u);
            uint32_t wm = __reduce_or_sync(0xffffffffu, m);
            while (wm) {
                const int b = 31 - __clz(wm);
                wm &= ~(1u << b);
                const int j = e0 + b - lo;
                const bool mine = (m >> b) & 1u;
                double v[9];
#pragma unroll
                for (int q = 0; q < 9; ++q) v[q] = 0.0;
                if (mine) {
                    const double mx = sh.f[0][j], my = sh.f[1][j], a = sh.f[2][j], bb = sh.f[3][j], c = sh.f[4][j];
                    const double al = sh.f[5][j], cr = sh.f[6][j], cg = sh.f[7][j], cb = sh.f[8][j];
                    // _composite.pyx:121-151, op for op
                    const double dy = pyd - my;
                    const double dx = pxd - mx;
                    const double e = 0.5 * (a * dx * dx + c * dy * dy) + bb * dx * dy;
                    const double gg = exp_tab(-e, exp_lane_tab(sh.exptab));
                    const double raw = al * gg;
                    const double ap = raw > kAlphaClamp ? kAlphaClamp : raw;
                    const double t_before = T / (1.0 - ap);
                    const double wgt = ap * t_before;
                    v[6] = wgt * dc0;
                    v[7] = wgt * dc1;
                    v[8] = wgt * dc2;
                    const double dc_dot_col = (dc0 * cr + dc1 * cg) + dc2 * cb;
                    double d_ap = t_before * dc_dot_col - ((ac0 * dc0 + ac1 * dc1) + ac2 * dc2) / (1.0 - ap);
                    if (raw >= kAlphaClamp) d_ap = 0.0;
                    v[5] = d_ap * gg;
                    const double d_g = d_ap * al;
                    const double d_e = -gg * d_g;
                    v[0] = -d_e * (a * dx + bb * dy);
                    v[1] = -d_e * (bb * dx + c * dy);
                    v[2] = d_e * 0.5 * dx * dx;
                    v[3] = d_e * dx * dy;
                    v[4] = d_e * 0.5 * dy * dy;
                    ac0 += cr * wgt;
                    ac1 += cg * wgt;
                    ac2 += cb * wgt;
                    T = t_before;
                }
                const unsigned who = __ballot_sync(0xffffffffu, mine);
                if (__popc(who) <= 2) {  // few contributors: their own reductions
                    if (mine)
#pragma unroll
                        for (int q = 0; q < 9; ++q) atomicAdd(G + (int64_t)sh.gid[j] * 9 + q, v[q]);
                } else {
#pragma unroll
                    for (int q = 0; q < 9; ++q) v[q] = warp_reduce_sum(v[q]);
                    if (lane == 0)
#pragma unroll
                        for (int q = 0; q < 9; ++q) atomicAdd(G + (int64_t)sh.gid[j] * 9 + q, v[q]);
                }
            }
        }

    }
}

struct ProjBwdArgs {
    airgs_frame fr;
    airgs_camera cam;
    const double *G;    // [n][9] image-space gradients per primitive
    double *grads;      // [n][W] row-major parameter gradients (written for every primitive)
};

// The chain rule of render_backward (ss/rasterizer.py:288-368), one thread per
// primitive; the forward quantities are recomputed with k_project's exact
// arithmetic.
template <int WMAX>
__global__ void __launch_bounds__(128) k_project_bwd(ProjBwdArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.fr.count) return;
    const int W = a.fr.width;
    const int64_t ld = a.fr.ld;
    double *gr = a.grads + i * W;
    for (int c = 0; c < W; ++c) gr[c] = 0.0;
    double Gv[9];
    bool any = false;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        Gv[q] = a.G[i * 9 + q];
        any |= Gv[q] != 0.0;
    }
    if (!any) return;  // not kept, or no recorded contribution: every term is zero
    double p[26];
#pragma unroll
    for (int c = 0; c < 26; ++c) p[c] = (c < W && c < WMAX) ? a.fr.params[i + c * ld] : 0.0;
    const airgs_camera &cam = a.cam;
    const double *R = cam.rot;
    const double f = cam.focal;
    // activation (ss/rasterizer.py:100-110)
    const double qn = sqrt(((p[3] * p[3] + p[4] * p[4]) + p[5] * p[5]) + p[6] * p[6]);
    const double qw = p[3] / qn, qx = p[4] / qn, qy = p[5] / qn, qz = p[6] / qn;
    const double s2v[3] = {exp(2.0 * p[7]), exp(2.0 * p[8]), exp(2.0 * p[9])};
    const double alpha = sigmoid_ref(p[10]);
    double rq[9];
    rq[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
    rq[1] = 2.0 * (qx * qy - qw * qz);
    rq[2] = 2.0 * (qx * qz + qw * qy);
    rq[3] = 2.0 * (qx * qy + qw * qz);
    rq[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
    rq[5] = 2.0 * (qy * qz - qw * qx);
    rq[6] = 2.0 * (qx * qz - qw * qy);
    rq[7] = 2.0 * (qy * qz + qw * qx);
    rq[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
    double cv[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            cv[3 * r + c] = dot3_blas(rq[3 * r] * s2v[0], rq[3 * r + 1] * s2v[1], rq[3 * r + 2] * s2v[2], rq[3 * c],
                                      rq[3 * c + 1], rq[3 * c + 2]);
    const double tx = dot3_blas(p[0], p[1], p[2], R[0], R[1], R[2]) + cam.trans[0];
    const double ty = dot3_blas(p[0], p[1], p[2], R[3], R[4], R[5]) + cam.trans[1];
    const double tz = dot3_blas(p[0], p[1], p[2], R[6], R[7], R[8]) + cam.trans[2];
    const double j00 = f / tz, zz = tz * tz, j02 = -f * tx / zz, j12 = -f * ty / zz;
    double M[6];
    for (int c = 0; c < 3; ++c) {
        M[c] = dot3_blas(j00, 0.0, j02, R[c], R[3 + c], R[6 + c]);
        M[3 + c] = dot3_blas(0.0, j00, j12, R[c], R[3 + c], R[6 + c]);
    }
    double MC[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            MC[3 * r + c] = dot3_blas(M[3 * r], M[3 * r + 1], M[3 * r + 2], cv[c], cv[3 + c], cv[6 + c]);
    const double a2 = dot3_blas(MC[0], MC[1], MC[2], M[0], M[1], M[2]) + kCovBlur;
    const double b2 = dot3_blas(MC[0], MC[1], MC[2], M[3], M[4], M[5]);
    const double c2 = dot3_blas(MC[3], MC[4], MC[5], M[3], M[4], M[5]) + kCovBlur;
    const double det = a2 * c2 - b2 * b2;
    const double ca = c2 / det, cbn = -b2 / det, cc = a2 / det;
    // d_cov2d = -conic @ g_full @ conic
    const double g00 = Gv[2], g01 = 0.5 * Gv[3], g11 = Gv[4];
    const double t00 = ca * g00 + cbn * g01, t01 = ca * g01 + cbn * g11;
    const double t10 = cbn * g00 + cc * g01, t11 = cbn * g01 + cc * g11;
    const double dc00 = -(t00 * ca + t01 * cbn), dc01 = -(t00 * cbn + t01 * cc);
    const double dc10 = -(t10 * ca + t11 * cbn), dc11 = -(t10 * cbn + t11 * cc);
    // d_m = 2 d_cov2d @ m @ cov3d ; d_cov3d = m^T d_cov2d m
    double DM[6], MCv[6];
    for (int c = 0; c < 3; ++c) {
        DM[c] = dc00 * M[c] + dc01 * M[3 + c];
        DM[3 + c] = dc10 * M[c] + dc11 * M[3 + c];
    }
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            MCv[3 * r + c] = 2.0 * ((DM[3 * r] * cv[c] + DM[3 * r + 1] * cv[3 + c]) + DM[3 * r + 2] * cv[6 + c]);
    double dcv[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            dcv[3 * r + c] = M[r] * DM[c] + M[3 + r] * DM[3 + c];
    // d_jac = d_m @ rot_wc^T
    double dj[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            dj[3 * r + c] = (MCv[3 * r] * R[3 * c] + MCv[3 * r + 1] * R[3 * c + 1]) + MCv[3 * r + 2] * R[3 * c + 2];
    const double inv_z = 1.0 / tz, inv_z2 = inv_z * inv_z;
    double dt0 = dj[2] * (-f * inv_z2);
    double dt1 = dj[5] * (-f * inv_z2);
    double dt2 = ((dj[0] * (-f * inv_z2) + dj[4] * (-f * inv_z2)) + dj[2] * (2 * f * tx * inv_z2 * inv_z)) +
                 dj[5] * (2 * f * ty * inv_z2 * inv_z);
    const double du = Gv[0], dv = Gv[1];
    dt0 += du * f * inv_z;
    dt1 += dv * f * inv_z;
    dt2 += -f * (du * tx + dv * ty) * inv_z2;
    double gpos[3];
    for (int k = 0; k < 3; ++k) gpos[k] = (R[k] * dt0 + R[3 + k] * dt1) + R[6 + k] * dt2;  // rot_wc^T d_t
    // scales and rotation through the 3D covariance
    double ps[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) ps[3 * r + c] = 0.5 * (dcv[3 * r + c] + dcv[3 * c + r]);
    for (int k = 0; k < 3; ++k) {
        const double r0 = rq[k], r1 = rq[3 + k], r2 = rq[6 + k];  // column k
        const double v0 = ps[0] * r0 + ps[1] * r1 + ps[2] * r2;
        const double v1 = ps[3] * r0 + ps[4] * r1 + ps[5] * r2;
        const double v2 = ps[6] * r0 + ps[7] * r1 + ps[8] * r2;
        gr[7 + k] += 2.0 * s2v[k] * ((r0 * v0 + r1 * v1) + r2 * v2);
    }
    double drot[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            drot[3 * r + c] = 2.0 * ((ps[3 * r] * rq[c] + ps[3 * r + 1] * rq[3 + c]) + ps[3 * r + 2] * rq[6 + c]) *
                              s2v[c];
    // _rot_jacobians (ss/rasterizer.py:262-268)
    const double Jw[9] = {0, -qz, qy, qz, 0, -qx, -qy, qx, 0};
    const double Jx[9] = {0, qy, qz, qy, -2 * qx, -qw, qz, qw, -2 * qx};
    const double Jy[9] = {-2 * qy, qx, qw, qx, 0, qz, -qw, qz, -2 * qy};
    const double Jz[9] = {-2 * qz, -qw, qx, qw, -2 * qz, qy, qx, qy, 0};
    double dq[4] = {0, 0, 0, 0};
    for (int k = 0; k < 9; ++k) {
        dq[0] += drot[k] * (2.0 * Jw[k]);
        dq[1] += drot[k] * (2.0 * Jx[k]);
        dq[2] += drot[k] * (2.0 * Jy[k]);
        dq[3] += drot[k] * (2.0 * Jz[k]);
    }
    const double qv[4] = {qw, qx, qy, qz};
    const double dqq = ((dq[0] * qw + dq[1] * qx) + dq[2] * qy) + dq[3] * qz;
    for (int k = 0; k < 4; ++k) gr[3 + k] += (dq[k] - dqq * qv[k]) / qn;
    // opacity logit
    gr[10] += Gv[5] * alpha * (1.0 - alpha);
    // colour logit and SH
    const double d0 = p[0] - cam.center[0], d1 = p[1] - cam.center[1], d2 = p[2] - cam.center[2];
    double dn = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    if (dn == 0.0) dn = 1.0;
    const double h0 = d0 / dn, h1 = d1 / dn, h2 = d2 / dn;
    double dl[3];
    for (int ch = 0; ch < 3; ++ch) {
        double lin = p[11 + ch] + kShC0 * p[14 + ch];
        if (WMAX == 26 && W == 26)
            lin = lin + kShC1 * ((-h1 * p[17 + ch] + h2 * p[20 + ch]) - h0 * p[23 + ch]);
        const double col = sigmoid_ref(lin);
        dl[ch] = Gv[6 + ch] * col * (1.0 - col);
        gr[11 + ch] += dl[ch];
        gr[14 + ch] += kShC0 * dl[ch];
    }
    if (WMAX == 26 && W == 26) {
        double dd[3] = {0, 0, 0};
        for (int ch = 0; ch < 3; ++ch) {
            gr[17 + ch] += -kShC1 * h1 * dl[ch];
            gr[20 + ch] += kShC1 * h2 * dl[ch];
            gr[23 + ch] += -kShC1 * h0 * dl[ch];
            // sh_block[coeff][ch] = params[17 + 3 coeff + ch]
            dd[0] += dl[ch] * (-kShC1 * p[23 + ch]);
            dd[1] += dl[ch] * (-kShC1 * p[17 + ch]);
            dd[2] += dl[ch] * (kShC1 * p[20 + ch]);
        }
        const double ddh = (dd[0] * h0 + dd[1] * h1) + dd[2] * h2;
        gpos[0] += (dd[0] - ddh * h0) / dn;
        gpos[1] += (dd[1] - ddh * h1) / dn;
        gpos[2] += (dd[2] - ddh * h2) / dn;
    }
    for (int k = 0; k < 3; ++k) gr[k] += gpos[k];
}

static void render_backward_impl(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                 const int64_t *frozen_pos, const double *d_image, double *grads,
                                 cudaStream_t st) {
    if (frame->count <= 0) throw ApiFailure(AIRGS_E_STRUCTURAL, "cannot render an empty frame");
    BwdState bw;
    bw.t_final = ctx->scratch_t<double>(kSlotTFinal, (size_t)cam->width * cam->height);
    airgs_view_item it{};
    it.frame = 0;
    it.camera = 0;
    it.frozen_pos = frozen_pos;
    // recompute the forward with its contribution record (deterministic: the same
    // lists, masks and final transmittance as render_forward)
    render_impl(ctx, frame, 1, cam, 1, &it, 1, nullptr, st, &bw);
    const int64_t n = frame->count;
    double *G = ctx->scratch_t<double>(kSlotBwdGrad, (size_t)n * 9);
    AIRGS_CUDA_TRY(cudaMemsetAsync(G, 0, sizeof(double) * 9 * n, st));
    if (bw.Tt > 0 && bw.rec.cbits) {
        const int tiles_x = (cam->width + kTile - 1) / kTile;
        k_composite_bwd<<<(unsigned)bw.Tt, kTileThreads, 0, st>>>(bw.recs, bw.rec.tl, bw.tile_count, bw.rec.cbits,
                                                                 bw.rec.cbase, tiles_x, cam->width, cam->height,
                                                                 bw.t_final, d_image, G);
        ++ctx->launches;
        check_launch();
    }
    ProjBwdArgs pa{*frame, *cam, G, grads};
    if (frame->width == 17)
        k_project_bwd<17><<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pa);
    else
        k_project_bwd<26><<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pa);
    ++ctx->launches;
    check_launch();
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
}

// Keep test and order key per primitive for one view, with k_project's exact
// arithmetic (ss/rasterizer.py:116-142): kept = z > near_clip and alpha > 1/255;
// key = order_key_of(frozen, i, z) for kept primitives, all ones otherwise.
__global__ void __launch_bounds__(256) k_order_keys(airgs_frame fr, airgs_camera cam, const int64_t *frozen,
                                                    uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                                                    unsigned long long *__restrict__ kept) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    uint64_t key = ~0ull;
    if (i < fr.count) {
        const int64_t ld = fr.ld;
        double p[11];
#pragma unroll
        for (int c = 0; c < 11; ++c) p[c] = fr.params[i + c * ld];
        const double alpha = sigmoid_ref(p[10]);
        const double *R = cam.rot;
        const double tz = dot3_blas(p[0], p[1], p[2], R[6], R[7], R[8]) + cam.trans[2];
        keep = tz > cam.near_clip && alpha > kEpsContrib;
        if (keep) key = order_key_of(frozen, i, tz);
        keys[i] = key;
        vals[i] = (uint32_t)i;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(kept, (unsigned long long)__popc(m));
}

__global__ void k_vals_to_order(const uint32_t *__restrict__ vals, int64_t n, int64_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = vals[i];
}

static void compositing_order_impl(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                   const int64_t *frozen_pos, int64_t *order_out, int64_t *kept_out,
                                   cudaStream_t st) {
    const int64_t n = frame->count;
    if (n <= 0) throw ApiFailure(AIRGS_E_STRUCTURAL, "cannot render an empty frame");
    if (n > (int64_t)0xffffffffLL) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");
    int64_t &NL = ctx->launches;
    uint64_t *k1 = ctx->scratch_t<uint64_t>(kSlotKeys, (size_t)n);
    uint64_t *k2 = ctx->scratch_t<uint64_t>(kSlotKeysAlt, (size_t)n);
    uint32_t *v1 = ctx->scratch_t<uint32_t>(kSlotVals, (size_t)n);
    uint32_t *v2 = ctx->scratch_t<uint32_t>(kSlotValsAlt, (size_t)n);
    int64_t *misc = ctx->scratch_t<int64_t>(kSlotMisc3, 4);
    AIRGS_CUDA_TRY(cudaMemsetAsync(misc, 0, sizeof(int64_t) * 4, st));
    k_order_keys<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(*frame, *cam, frozen_pos, k1, v1,
                                                            (unsigned long long *)misc);
    ++NL;
    const int64_t seg[2] = {0, n};
    int64_t *d_seg = misc + 2;
    h2d_small(ctx, d_seg, seg, sizeof(seg), st);
    uint32_t *hist = ctx->scratch_t<uint32_t>(kSlotHist, (size_t)256 * ceil_div(n, kSortTile));
    // stable LSD radix sort on the 64-bit key; equal keys keep the index order
    const bool alt = radix_sort<uint64_t>(k1, v1, k2, v2, d_seg, d_seg + 1, 1, n, 64, hist, st, &NL);
    k_vals_to_order<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(alt ? v2 : v1, n, order_out);
    ++NL;
    check_launch();
    AIRGS_CUDA_TRY(cudaMemcpyAsync(kept_out, misc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
}

// ---- kernel seam record / backward: the reference's mask layout -----------
// masks[off_i + (iy - y0) * (x1 - x0) + (ix - x0)] for primitive i's clipped
// bbox, off_i = prefix of the non-empty bbox areas (ss/_composite.pyx:29-35,
// 67-73); tile bits <-> reference masks through the primitive's position in the
// tile list (sorted by input index on the seam).

__device__ __forceinline__ int list_find(const uint64_t *lst, int n, uint32_t id) {
    int lo = 0, hi = n - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t v = (uint32_t)lst[mid];
        if (v == id) return mid;
        if (v < id) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

// one block per primitive: its bbox pixels' contribution bits -> reference masks
__global__ void __launch_bounds__(128) k_masks_from_bits(const int64_t *__restrict__ bboxes,
                                                         const int64_t *__restrict__ moff, const TileLists tls,
                                                         const uint32_t *__restrict__ tcount,
                                                         const uint32_t *__restrict__ cbits,
                                                         const int64_t *__restrict__ cbase, int tiles_x,
                                                         uint8_t *__restrict__ masks) {
    const int64_t i = blockIdx.x;
    const int x0 = (int)bboxes[4 * i], x1 = (int)bboxes[4 * i + 1], y0 = (int)bboxes[4 * i + 2],
              y1 = (int)bboxes[4 * i + 3];
    if (x1 <= x0 || y1 <= y0) return;
    const int bw = x1 - x0;
    const int64_t area = (int64_t)bw * (y1 - y0);
    for (int64_t q = threadIdx.x; q < area; q += blockDim.x) {
        const int iy = y0 + (int)(q / bw), ix = x0 + (int)(q % bw);
        const int64_t g = (int64_t)(iy / kTile) * tiles_x + ix / kTile;
        const int e = list_find(tls.list(g), tls.count(tcount, g), (uint32_t)i);
        uint8_t m = 0;
        if (e >= 0)
            m = (cbits[cbase[g] + (int64_t)(e >> 5) * kTileThreads + (iy % kTile) * kTile + ix % kTile] >> (e & 31)) & 1u;
        masks[moff[i] + q] = m;
    }
}

// one block per tile: reference masks -> contribution bits of the tile's entries
__global__ void __launch_bounds__(kTileThreads) k_bits_from_masks(const int64_t *__restrict__ bboxes,
                                                                  const int64_t *__restrict__ moff,
                                                                  const TileLists tls,
                                                                  const uint32_t *__restrict__ tcount,
                                                                  const int64_t *__restrict__ cbase, int tiles_x,
                                                                  int w, int h, const uint8_t *__restrict__ masks,
                                                                  uint32_t *__restrict__ cbits) {
    const int64_t g = blockIdx.x;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int ix = (int)(g % tiles_x) * kTile + lx, iy = (int)(g / tiles_x) * kTile + ly;
    const int n = tls.count(tcount, g);
    const uint64_t *lst = tls.list(g);
    uint32_t word = 0;
    for (int e = 0; e < n; ++e) {
        const int64_t i = (uint32_t)lst[e];
        const int x0 = (int)bboxes[4 * i], x1 = (int)bboxes[4 * i + 1], y0 = (int)bboxes[4 * i + 2],
                  y1 = (int)bboxes[4 * i + 3];
        if (ix < w && iy < h && ix >= x0 && ix < x1 && iy >= y0 && iy < y1 &&
            masks[moff[i] + (int64_t)(iy - y0) * (x1 - x0) + (ix - x0)])
            word |= 1u << (e & 31);
        if ((e & 31) == 31 || e == n - 1) {
            cbits[cbase[g] + (int64_t)(e >> 5) * kTileThreads + threadIdx.x] = word;
            word = 0;
        }
    }
}

static void seam_impl(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics, const double *alphas,
                      const double *colors, const int64_t *bboxes, int h, int w, double *image, double *tfinal,
                      int64_t *usage, cudaStream_t st, RecordOut *rec = nullptr, Rec **recs_out = nullptr,
                      int64_t *Tt_out = nullptr, uint32_t **tcount_out = nullptr) {
    if (h < 1 || w < 1) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad image size");
    if (w > 65535 * kTile || h > 65535 * kTile) throw ApiFailure(AIRGS_E_CAPACITY, "image beyond the tile index range");
    if (k >= (1LL << 30)) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");  // list keys: index < 2^30
    std::vector<ItemHost> ih(1);
    ItemHost &it = ih[0];
    it.frame = 0;
    it.cam = 0;
    it.count = k;
    it.w = w;
    it.h = h;
    it.tiles_x = (w + kTile - 1) / kTile;
    it.tiles_y = (h + kTile - 1) / kTile;
    it.target = nullptr;
    it.image = image;
    it.trans = tfinal;
    it.usage = usage;
    it.clip = 0;
    Layout L;
    L.stride = std::max<int64_t>(k, 1);
    upload_layout(ctx, ih, L, st);
    Rec *recs = ctx->scratch_t<Rec>(kSlotRecs, L.stride);
    int32_t *ntiles = ctx->scratch_t<int32_t>(kSlotNtiles, L.stride);
    uint2 *binrec = ctx->scratch_t<uint2>(kSlotBinRec, L.stride);
    uint64_t *depth = ctx->scratch_t<uint64_t>(kSlotDepth, L.stride);
    uint32_t *tile_count = ctx->scratch_t<uint32_t>(kSlotTileCount, (size_t)L.Tt);
    AIRGS_CUDA_TRY(cudaMemsetAsync(tile_count, 0, sizeof(uint32_t) * L.Tt, st));
    unsigned int *flags = ctx->scratch_t<unsigned int>(kSlotFlags, 4);
    AIRGS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(unsigned int), st));
    if (usage && k > 0) AIRGS_CUDA_TRY(cudaMemsetAsync(usage, 0, sizeof(int64_t) * k, st));
    if (k > 0) {
        k_seam_records<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, means2d, conics, alphas, colors, bboxes, recs,
                                                                  ntiles, depth, binrec);
        ++ctx->launches;
        check_launch();
    }
    // every in-image pixel of every tile is written by the composite kernel
    bin_and_composite(ctx, ih, L, recs, depth, ntiles, tile_count, 1, nullptr, st, flags, binrec, nullptr, rec);
    if (recs_out) *recs_out = recs;
    if (Tt_out) *Tt_out = L.Tt;
    if (tcount_out) *tcount_out = tile_count;
}

// forward(record=True): the seam forward plus the reference's masks
static void seam_record_impl(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics,
                             const double *alphas, const double *colors, const int64_t *bboxes, int h, int w,
                             double *image, double *tfinal, int64_t *usage, const int64_t *moff, uint8_t *masks,
                             cudaStream_t st) {
    RecordOut rec;
    int64_t Tt = 0;
    uint32_t *tcount = nullptr;
    seam_impl(ctx, k, means2d, conics, alphas, colors, bboxes, h, w, image, tfinal, usage, st, &rec, nullptr, &Tt,
              &tcount);
    if (k > 0 && Tt > 0 && rec.cbits) {
        k_masks_from_bits<<<(unsigned)k, 128, 0, st>>>(bboxes, moff, rec.tl, tcount, rec.cbits, rec.cbase,
                                                       (w + kTile - 1) / kTile, masks);
        ++ctx->launches;
        check_launch();
    }
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
}

// backward(masks, t_final, d_image) of the seam (ss/_composite.pyx:77-152):
// grads9 = [k][d_means2d x, y, d_conics a, b, c, d_alphas, d_colors r, g, b]
static void seam_backward_impl(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics,
                               const double *alphas, const double *colors, const int64_t *bboxes, int h, int w,
                               const int64_t *moff, const uint8_t *masks, const double *tfinal,
                               const double *d_image, double *grads9, cudaStream_t st) {
    if (k > 0) AIRGS_CUDA_TRY(cudaMemsetAsync(grads9, 0, sizeof(double) * 9 * k, st));
    RecordOut rec;
    Rec *recs = nullptr;
    int64_t Tt = 0;
    uint32_t *tcount = nullptr;
    // the tile lists (and a record buffer of the right layout) from the seam pipeline
    seam_impl(ctx, k, means2d, conics, alphas, colors, bboxes, h, w, nullptr, nullptr, nullptr, st, &rec, &recs, &Tt,
              &tcount);
    if (k <= 0 || Tt <= 0 || !rec.cbits) return;
    const int tiles_x = (w + kTile - 1) / kTile;
    k_bits_from_masks<<<(unsigned)Tt, kTileThreads, 0, st>>>(bboxes, moff, rec.tl, tcount, rec.cbase, tiles_x, w, h,
                                                           masks, rec.cbits);
    k_composite_bwd<<<(unsigned)Tt, kTileThreads, 0, st>>>(recs, rec.tl, tcount, rec.cbits, rec.cbase, tiles_x, w, h,
                                                         tfinal, d_image, grads9);
    ctx->launches += 2;
    check_launch();
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
}

static void sse_impl(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *out, cudaStream_t st) {
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(1184, ceil_div(n, 4096)));
    double *part = ctx->scratch_t<double>(kSlotMisc0, parts);
    if (n > 0) {
        k_sse_flat_partial<<<parts, 256, 0, st>>>(a, b, n, part);
    } else {
        AIRGS_CUDA_TRY(cudaMemsetAsync(part, 0, sizeof(double), st));
    }
    k_sse_flat_final<<<1, 32, 0, st>>>(part, n > 0 ? parts : 1, out);
    ctx->launches += 2;
    check_launch();
}

}  // namespace airgs

using namespace airgs;

// ---------------------------------------------------------------------------
// tile footprint (pruning-level sweep, clean-tile skip; include/airgs_b200.h)

// The projection of k_project restated for the clipped bbox and the
// threshold-ellipse AABB alone (same fp64 expressions, so the same extents),
// each widened by a pixel or more: every tile the binning gives the primitive
// (clipped bbox ∩ threshold-ellipse AABB, rec_tile_range) is marked.
// Non-finite geometry marks the whole view.
__global__ void __launch_bounds__(128) k_tile_footprint(airgs_frame fr, const airgs_camera *__restrict__ cams,
                                                         int ncams, const int32_t *__restrict__ rank, int32_t rank_cap,
                                                         int32_t *__restrict__ minrank, int64_t tile_stride) {
    // one thread per primitive, its view-independent terms once, then every view
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= fr.count) return;
    const int32_t rk = rank[i];
    if (rk >= rank_cap) return;
    const int64_t ld = fr.ld;
    double p[11];
    bool finite = true;
#pragma unroll
    for (int c = 0; c < 11; ++c) {
        p[c] = fr.params[i + c * ld];
        finite &= isfinite(p[c]);
    }
    for (int c = 11; c < fr.width; ++c) finite &= isfinite(fr.params[i + c * ld]);
    const double qn = sqrt(((p[3] * p[3] + p[4] * p[4]) + p[5] * p[5]) + p[6] * p[6]);
    if (!finite || qn == 0.0) return;  // the render of this frame fails (ss/rasterizer.py:105-106)
    const double alpha = sigmoid_ref(p[10]);
    if (!(alpha > kEpsContrib * (1.0 - 1e-12))) return;  // not kept by either render
    const double w_ = p[3] / qn, x_ = p[4] / qn, y_ = p[5] / qn, z_ = p[6] / qn;
    const double s0 = exp(2.0 * p[7]), s1 = exp(2.0 * p[8]), s2 = exp(2.0 * p[9]);
    double m[9];
    m[0] = 1.0 - 2.0 * (y_ * y_ + z_ * z_);
    m[1] = 2.0 * (x_ * y_ - w_ * z_);
    m[2] = 2.0 * (x_ * z_ + w_ * y_);
    m[3] = 2.0 * (x_ * y_ + w_ * z_);
    m[4] = 1.0 - 2.0 * (x_ * x_ + z_ * z_);
    m[5] = 2.0 * (y_ * z_ - w_ * x_);
    m[6] = 2.0 * (x_ * z_ - w_ * y_);
    m[7] = 2.0 * (y_ * z_ + w_ * x_);
    m[8] = 1.0 - 2.0 * (x_ * x_ + y_ * y_);
    double cv[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            cv[3 * r + c] = dot3_blas(m[3 * r] * s0, m[3 * r + 1] * s1, m[3 * r + 2] * s2, m[3 * c], m[3 * c + 1],
                                      m[3 * c + 2]);
    const double t2 = 2.0 * fmax(log(alpha / kEpsContrib) * 1.0002 + 2e-4, 0.0);
    for (int v = 0; v < ncams; ++v) {
        const airgs_camera &cam = cams[v];
        const double *R = cam.rot;
        const double tz = dot3_blas(p[0], p[1], p[2], R[6], R[7], R[8]) + cam.trans[2];
        if (!(tz > cam.near_clip - 1e-9 * (1.0 + fabs(cam.near_clip)))) continue;
        const int txn = (cam.width + kTile - 1) / kTile, tyn = (cam.height + kTile - 1) / kTile;
        int32_t *mr = minrank + (int64_t)v * tile_stride;
        const double tx = dot3_blas(p[0], p[1], p[2], R[0], R[1], R[2]) + cam.trans[0];
        const double ty = dot3_blas(p[0], p[1], p[2], R[3], R[4], R[5]) + cam.trans[1];
        const double fl = cam.focal;
        const double mx = fl * tx / tz + 0.5 * (double)cam.width;
        const double my = fl * ty / tz + 0.5 * (double)cam.height;
        const double j00 = fl / tz, zz = tz * tz, j02 = -fl * tx / zz, j12 = -fl * ty / zz;
        double M[6];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            M[c] = dot3_blas(j00, 0.0, j02, R[c], R[3 + c], R[6 + c]);
            M[3 + c] = dot3_blas(0.0, j00, j12, R[c], R[3 + c], R[6 + c]);
        }
        double MC[6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                MC[3 * r + c] = dot3_blas(M[3 * r], M[3 * r + 1], M[3 * r + 2], cv[c], cv[3 + c], cv[6 + c]);
        const double a2 = dot3_blas(MC[0], MC[1], MC[2], M[0], M[1], M[2]) + kCovBlur;
        const double b2 = dot3_blas(MC[0], MC[1], MC[2], M[3], M[4], M[5]);
        const double c2 = dot3_blas(MC[3], MC[4], MC[5], M[3], M[4], M[5]) + kCovBlur;
        const double dd = a2 - c2;
        const double eig = 0.5 * (a2 + c2) + sqrt(fmax(0.25 * (dd * dd) + b2 * b2, 0.0));
        const double rad = kRadiusSigma * sqrt(eig);
        const double Wd = (double)cam.width, Hd = (double)cam.height;
        int u0 = 0, u1 = txn - 1, v0 = 0, v1 = tyn - 1;
        if (isfinite(mx) && isfinite(my) && isfinite(rad)) {
            const int x0 = (int)fmin(fmax(floor(mx - rad) - 1.0, 0.0), Wd);
            const int x1 = (int)fmin(fmax(ceil(mx + rad) + 2.0, 0.0), Wd);
            const int y0 = (int)fmin(fmax(floor(my - rad) - 1.0, 0.0), Hd);
            const int y1 = (int)fmin(fmax(ceil(my + rad) + 2.0, 0.0), Hd);
            if (x1 <= x0 || y1 <= y0) continue;
            int xa = x0, xb = x1 - 1, ya = y0, yb = y1 - 1;
            const double det = a2 * c2 - b2 * b2;
            const double hx = sqrt(t2 * (a2 + 1e-9 * a2)) * 1.0002 + 1e-3;
            const double hy = sqrt(t2 * (c2 + 1e-9 * c2)) * 1.0002 + 1e-3;
            if (det > 0.0 && isfinite(hx) && isfinite(hy)) {  // k_project's rec.hx / rec.hy, padded outward
                const double ex = hx * 1.001 + 2.0, ey = hy * 1.001 + 2.0;
                xa = max(xa, (int)fmax(floor(mx - 0.5 - ex), -1.0));
                xb = min(xb, (int)fmin(ceil(mx - 0.5 + ex), Wd));
                ya = max(ya, (int)fmax(floor(my - 0.5 - ey), -1.0));
                yb = min(yb, (int)fmin(ceil(my - 0.5 + ey), Hd));
                if (xa > xb || ya > yb) continue;
            }
            u0 = xa / kTile;
            u1 = xb / kTile;
            v0 = ya / kTile;
            v1 = yb / kTile;
        }
        for (int y = v0; y <= v1; ++y)
            for (int x = u0; x <= u1; ++x) {
                int32_t *q = mr + (int64_t)y * txn + x;
                if (*q > rk) atomicMin(q, rk);
            }
    }
}

static void tile_footprint_impl(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cams, int ncams,
                                const int32_t *rank, int32_t rank_cap, int32_t *minrank, int64_t tile_stride,
                                cudaStream_t st) {
    if (ncams <= 0 || frame->count <= 0 || rank_cap <= 0) return;
    if (frame->width != 17 && frame->width != 26)
        throw ApiFailure(AIRGS_E_STRUCTURAL, "no sh degree yields parameter width " + std::to_string(frame->width));
    for (int v = 0; v < ncams; ++v) {
        const airgs_camera &c = cams[v];
        if (c.width < 1 || c.height < 1) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad camera resolution");
        if (ceil_div(c.width, kTile) * ceil_div(c.height, kTile) > tile_stride)
            throw ApiFailure(AIRGS_E_CAPACITY, "tile_stride below a camera's tile count");
    }
    airgs_camera *d_cams = ctx->scratch_t<airgs_camera>(kSlotMisc1, (size_t)ncams);
    h2d_small(ctx, d_cams, cams, sizeof(airgs_camera) * ncams, st);
    k_tile_footprint<<<(unsigned)ceil_div(frame->count, 128), 128, 0, st>>>(*frame, d_cams, ncams, rank, rank_cap,
                                                                            minrank, tile_stride);
    ++ctx->launches;
    check_launch();
}

extern "C" int airgs_tile_footprint(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cams, int32_t ncams,
                                    const int32_t *rank, int32_t rank_cap, int32_t *minrank, int64_t tile_stride,
                                    void *stream) {
    return guarded(ctx, [&] {
        tile_footprint_impl(ctx, frame, cams, ncams, rank, rank_cap, minrank, tile_stride, (cudaStream_t)stream);
    });
}

extern "C" int airgs_render(airgs_ctx *ctx, const airgs_frame *frames, int32_t nframes, const airgs_camera *cams,
                            int32_t ncams, const airgs_view_item *items, int32_t nitems, double *sse, void *stream) {
    return guarded(ctx, [&] { render_impl(ctx, frames, nframes, cams, ncams, items, nitems, sse, (cudaStream_t)stream); });
}

#ifdef C2_COUNT
extern "C" __attribute__((visibility("default"))) int airgs_c2_counts(unsigned long long *out, int reset) {
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(out, g_c2c, sizeof(unsigned long long) * 10) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[10] = {};
        cudaMemcpyToSymbol(g_c2c, z, sizeof(z));
    }
    return 0;
}
#endif

extern "C" int airgs_debug_tile_lists(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                      int64_t max_per_tile, int32_t *counts, int32_t *ids, void *stream) {
    return guarded(ctx, [&] {
        if (max_per_tile <= 0 || !counts || !ids) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad tile dump buffers");
        struct Reset {
            airgs_ctx *c;
            ~Reset() { c->dump = airgs_ctx::TileDump{}; }
        } reset{ctx};
        ctx->dump.counts = counts;
        ctx->dump.ids = ids;
        ctx->dump.max_per_tile = max_per_tile;
        airgs_view_item it{0, 0, nullptr, nullptr, nullptr, nullptr};
        const bool deferred = ctx->defer;
        ctx->defer = false;  // checked call: an overflowing bucket is redone through scanned ranges
        try {
            render_impl(ctx, frame, 1, cam, 1, &it, 1, nullptr, (cudaStream_t)stream);
        } catch (...) {
            ctx->defer = deferred;
            throw;
        }
        ctx->defer = deferred;
        AIRGS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    });
}

extern "C" int airgs_composite_forward(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics,
                                       const double *alphas, const double *colors, const int64_t *bboxes,
                                       int32_t height, int32_t width, double *image, double *t_final,
                                       int64_t *usage, void *stream) {
    return guarded(ctx, [&] {
        seam_impl(ctx, k, means2d, conics, alphas, colors, bboxes, height, width, image, t_final, usage,
                  (cudaStream_t)stream);
    });
}

extern "C" int airgs_render_backward(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                     const int64_t *frozen_pos, const double *d_image, double *grads,
                                     void *stream) {
    return guarded(ctx, [&] {
        render_backward_impl(ctx, frame, cam, frozen_pos, d_image, grads, (cudaStream_t)stream);
    });
}

extern "C" int airgs_compositing_order(airgs_ctx *ctx, const airgs_frame *frame, const airgs_camera *cam,
                                       const int64_t *frozen_pos, int64_t *order_out, int64_t *kept_out,
                                       void *stream) {
    return guarded(ctx, [&] {
        compositing_order_impl(ctx, frame, cam, frozen_pos, order_out, kept_out, (cudaStream_t)stream);
    });
}

extern "C" int airgs_composite_forward_record(airgs_ctx *ctx, int64_t k, const double *means2d,
                                              const double *conics, const double *alphas, const double *colors,
                                              const int64_t *bboxes, int32_t height, int32_t width, double *image,
                                              double *t_final, int64_t *usage, const int64_t *mask_offsets,
                                              uint8_t *masks, void *stream) {
    return guarded(ctx, [&] {
        seam_record_impl(ctx, k, means2d, conics, alphas, colors, bboxes, height, width, image, t_final, usage,
                         mask_offsets, masks, (cudaStream_t)stream);
    });
}

extern "C" int airgs_composite_backward(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics,
                                        const double *alphas, const double *colors, const int64_t *bboxes,
                                        int32_t height, int32_t width, const int64_t *mask_offsets,
                                        const uint8_t *masks, const double *t_final, const double *d_image,
                                        double *grads9, void *stream) {
    return guarded(ctx, [&] {
        seam_backward_impl(ctx, k, means2d, conics, alphas, colors, bboxes, height, width, mask_offsets, masks,
                           t_final, d_image, grads9, (cudaStream_t)stream);
    });
}

extern "C" int airgs_sse(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *out, void *stream) {
    return guarded(ctx, [&] { sse_impl(ctx, a, b, n, out, (cudaStream_t)stream); });
}
