// Batched rasterizer for the AirGS evaluation path on B200 (sm_100a).
//
// Pipeline per batch of view items (frame, camera):
//   k_project       fp64 activation + EWA projection, op-for-op with
//                   ss/rasterizer.py:100-212 (one thread per primitive, all
//                   views of its frame in the inner loop so the parameter row
//                   and the view-independent activation are read/computed once)
//   compaction      stable per-item scan of visible primitives (warp scans)
//   depth sort      stable LSD radix sort of (z bits - zmin) -> depth rank;
//                   ties keep index order == np.argsort(kind="stable")
//   binning         (tile) keys emitted in rank order, stable radix sort by
//                   tile -> per-tile lists in depth order
//   k_composite     16x16 tile per CTA, one pixel per thread, front-to-back
//                   with exact early termination; fp32 log-domain fast reject
//                   with a proven guard band, exact fp64 replay of
//                   _composite.pyx:42-73 for every surviving (pixel, primitive)
//                   pair; fused usage counts and per-tile SSE
//   k_sse_items     deterministic per-item SSE reduction
#include <algorithm>
#include <cmath>
#include <vector>

#include "context.h"
#include "exp_table.h"
#include "scan_sort.cuh"

namespace airgs {

// ---------------------------------------------------------------------------
// projection

struct ProjArgs {
    const airgs_frame *frames;
    const airgs_camera *cams;
    const int32_t *frame_item_ptr;  // CSR over frames
    const int32_t *frame_items;
    const int32_t *item_cam;
    Rec *recs;                 // [nitems][stride]
    uint64_t *depth;           // [nitems][stride]
    int32_t *ntiles;           // [nitems][stride]
    unsigned long long *zmin;  // [nitems]
    unsigned long long *zmax;  // [nitems]
    unsigned int *flags;
    int64_t stride;
};

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

constexpr int kProjThreads = 128;

__global__ void __launch_bounds__(kProjThreads) k_project(ProjArgs a) {
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
    for (int c = 0; c < 26; ++c) p[c] = (active && c < W) ? fr.params[i + c * ld] : 0.0;

    // _activate (ss/rasterizer.py:100-110)
    const double qn = sqrt(((p[3] * p[3] + p[4] * p[4]) + p[5] * p[5]) + p[6] * p[6]);
    bool finite = true;
#pragma unroll
    for (int c = 0; c < 26; ++c) finite &= isfinite(p[c]);
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
    // SH degree 0: colour is view independent -- compute once
    double col0[3] = {0.0, 0.0, 0.0};
    if (W == 17 && live) {
        col0[0] = sigmoid_ref(p[11] + kShC0 * p[14]);
        col0[1] = sigmoid_ref(p[12] + kShC0 * p[15]);
        col0[2] = sigmoid_ref(p[13] + kShC0 * p[16]);
    }
    __shared__ unsigned long long red_min[kProjThreads / 32], red_max[kProjThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    for (int it = ib; it < ie; ++it) {
        const int item = a.frame_items[it];
        const int64_t o = (int64_t)item * a.stride + i;
        const airgs_camera &cam = a.cams[a.item_cam[item]];
        const double *R = cam.rot;
        unsigned long long zkey_min = ~0ull, zkey_max = 0ull;
        int nt = 0;
        double tz = 0.0;
        if (live) tz = dot3_blas(p[0], p[1], p[2], R[6], R[7], R[8]) + cam.trans[2];
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
            rec.x0 = (int32_t)fmin(fmax(floor(mx - rad), 0.0), Wd);
            rec.x1 = (int32_t)fmin(fmax(ceil(mx + rad) + 1.0, 0.0), Wd);
            rec.y0 = (int32_t)fmin(fmax(floor(my - rad), 0.0), Hd);
            rec.y1 = (int32_t)fmin(fmax(ceil(my + rad) + 1.0, 0.0), Hd);
            if (W == 26) {  // colour (ss/rasterizer.py:183-198), view dependent
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
                const double t = log(alpha / kEpsContrib) * 1.0002 + 2e-4;
                const double hx = sqrt(2.0 * fmax(t, 0.0) * (a2 + 1e-9 * a2)) * 1.0002 + 1e-3;
                const double hy = sqrt(2.0 * fmax(t, 0.0) * (c2 + 1e-9 * c2)) * 1.0002 + 1e-3;
                rec.hx = det > 0.0 && isfinite(hx) ? (float)hx * 1.0001f : 1e30f;
                rec.hy = det > 0.0 && isfinite(hy) ? (float)hy * 1.0001f : 1e30f;
            }
            if (rec.x1 > rec.x0 && rec.y1 > rec.y0)
                nt = ((rec.x1 - 1) / kTile - rec.x0 / kTile + 1) * ((rec.y1 - 1) / kTile - rec.y0 / kTile + 1);
            if (nt > 0) {
                a.recs[o] = rec;
                const unsigned long long zk = order_key(tz);
                a.depth[o] = zk;
                zkey_min = zkey_max = zk;
            }
        }
        if (active) a.ntiles[o] = nt;
        // block-level min/max of the depth keys -> one atomic pair per block
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            zkey_min = min(zkey_min, __shfl_xor_sync(0xffffffffu, zkey_min, d));
            zkey_max = max(zkey_max, __shfl_xor_sync(0xffffffffu, zkey_max, d));
        }
        if (lane == 0) {
            red_min[wid] = zkey_min;
            red_max[wid] = zkey_max;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long mn = red_min[0], mxk = red_max[0];
            for (int k = 1; k < kProjThreads / 32; ++k) {
                mn = min(mn, red_min[k]);
                mxk = max(mxk, red_max[k]);
            }
            if (mxk) {
                atomicMin(a.zmin + item, mn);
                atomicMax(a.zmax + item, mxk);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// scan functors

struct VisIn {
    const int32_t *nt;
    int64_t stride;
    __device__ int64_t operator()(int s, int64_t i) const { return nt[(int64_t)s * stride + i] > 0 ? 1 : 0; }
};
struct VisOut {
    const uint64_t *depth;
    const unsigned long long *zmin;
    uint64_t *keys;
    uint32_t *vals;
    int64_t stride;
    __device__ void operator()(int s, int64_t i, int64_t ex, int64_t v) const {
        if (v) {
            const int64_t b = (int64_t)s * stride;
            keys[b + ex] = depth[b + i] - zmin[s];
            vals[b + ex] = (uint32_t)i;
        }
    }
};
struct TileCountIn {
    const int32_t *nt;
    const uint32_t *vals;
    int64_t stride;
    __device__ int64_t operator()(int s, int64_t r) const {
        const int64_t b = (int64_t)s * stride;
        return nt[b + vals[b + r]];
    }
};
struct TileCountOut {
    int64_t *off;
    int64_t stride;
    __device__ void operator()(int s, int64_t r, int64_t ex, int64_t) const {
        off[(int64_t)s * stride + r] = ex;
    }
};

// ---------------------------------------------------------------------------
// binning

struct EmitArgs {
    const Rec *recs;
    const uint32_t *vals;      // rank -> primitive per item
    const int64_t *pair_off;   // rank -> offset within item's pairs
    const int64_t *nvis;       // per item
    const int64_t *pair_begin; // per item
    const int32_t *tiles_x;    // per item
    uint32_t *pkeys;
    uint32_t *pvals;
    int64_t stride;
};

__global__ void __launch_bounds__(256) k_emit_pairs(EmitArgs a) {
    const int s = blockIdx.y;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.nvis[s]) return;
    const int64_t b = (int64_t)s * a.stride;
    const uint32_t i = a.vals[b + r];
    const Rec &rec = a.recs[b + i];
    const int tx = a.tiles_x[s];
    int64_t o = a.pair_begin[s] + a.pair_off[b + r];
    const int u0 = rec.x0 / kTile, u1 = (rec.x1 - 1) / kTile;
    const int v0 = rec.y0 / kTile, v1 = (rec.y1 - 1) / kTile;
    for (int v = v0; v <= v1; ++v)
        for (int u = u0; u <= u1; ++u) {
            a.pkeys[o] = (uint32_t)(v * tx + u);
            a.pvals[o] = i;
            ++o;
        }
}

__global__ void __launch_bounds__(256)
k_tile_ranges(const uint32_t *__restrict__ pkeys, const int64_t *__restrict__ pair_begin,
              const int64_t *__restrict__ npairs, const int64_t *__restrict__ tile_base,
              int64_t *__restrict__ tstart, int64_t *__restrict__ tend) {
    const int s = blockIdx.y;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = npairs[s];
    if (r >= n) return;
    const uint32_t *k = pkeys + pair_begin[s];
    const uint32_t key = k[r];
    const int64_t g = tile_base[s] + key;
    if (r == 0 || k[r - 1] != key) tstart[g] = r;
    if (r == n - 1 || k[r + 1] != key) tend[g] = r + 1;
}

// ---------------------------------------------------------------------------
// compositing

struct CompItem {
    const Rec *recs;         // primitive records of this item
    const uint32_t *gids;    // sorted pair values (primitive ids) of this item
    const int64_t *tstart;   // per tile of this item
    const int64_t *tend;
    const double *target;    // (h,w,3) or null
    double *image;           // (h,w,3) or null
    double *trans;           // (h,w) or null
    int64_t *usage;          // [n] or null
    double *sse_tiles;       // per tile of this item
    int32_t w, h, tiles_x, clip;
};

constexpr double kLog2e = 1.4426950408889634;
// log2(1 / fl(1/255)) rounded to fp32 (threshold offset in the log2 domain)
__device__ __forceinline__ float log2_inv_eps() { return 7.99435343685886f; }

// exp(x) for the compositing weights: 256-entry table of 2^(i/256) in shared
// memory + degree-5 polynomial on |r| <= ln2/512 (error < 0.51 ulp; agrees
// with glibc's exp, which the reference's Cython kernel calls, on >99.9% of
// inputs and never differs by more than 1 ulp -- tools/gen_exp_table.py).
__device__ __forceinline__ double exp_tab(double x, const double2 *__restrict__ tab) {
    const double shift = 6755399441055744.0;  // 1.5 * 2^52
    const double z = x * kExpInvLn2N;
    double kd = z + shift;
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = kd - shift;
    double r = fma(kd, kExpNegLn2HiN, x);
    r = fma(kd, kExpNegLn2LoN, r);
    const double2 t = tab[ki & (kExpN - 1)];
    const unsigned long long sb = (unsigned long long)__double_as_longlong(t.y) + (ki << (52 - kExpBits));
    const double r2 = r * r;
    const double p1 = fma(r, 1.0 / 6.0, 0.5);
    const double p2 = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    double tmp = t.x + r;
    tmp = fma(r2, p1, tmp);
    tmp = fma(r2 * r2, p2, tmp);
    const double sc = __longlong_as_double((long long)sb);
    return fma(sc, tmp, sc);
}

struct CompShared {
    float4 f0[kTileThreads];     // mx-ox, my-oy (tile origin), 0.5*log2e*a, log2e*b  (fp32, log2 domain)
    float2 f1[kTileThreads];     // 0.5*log2e*c, log2(alpha)
    double2 m[kTileThreads];     // mx, my
    double2 hab[kTileThreads];   // 0.5*a, b
    double2 hcal[kTileThreads];  // 0.5*c, alpha
    double2 rg[kTileThreads];    // colour r, g
    double bl[kTileThreads];     // colour b
    uint32_t gid[kTileThreads];
    int32_t cnt[kTileThreads];
    uint8_t wmask[kTileThreads];  // bit w: may touch warp w's 8x4 sub-tile
    double2 exptab[kExpN];
};

constexpr int kCompWarps = kTileThreads / 32;
#ifndef COMP_MIN_BLOCKS
#define COMP_MIN_BLOCKS 3
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
    const double ap = ca.y * exp_tab(-ee, sh.exptab);
    return ap > kAlphaClamp ? kAlphaClamp : ap;
}

// One CTA = one 16x16 tile, one pixel per thread; warps are 8x4 sub-tiles.
// Per batch of 256 depth-ordered primitives (staged once per CTA), each warp
// walks 32-entry chunks: phase A tests only primitives whose threshold-ellipse
// AABB touches its sub-tile (fp32, log2 domain, proven guard band) and builds
// a per-lane candidate mask; phase B has every lane run its own candidates
// through the exact fp64 path in depth order (two candidates' exp in flight).
template <bool USAGE>
__global__ void __launch_bounds__(kTileThreads, COMP_MIN_BLOCKS)
k_composite(const CompItem *__restrict__ items, const int64_t *__restrict__ tile_base, int nitems) {
    __shared__ CompShared sh;
    {
        const unsigned long long *src = &kExpTable[0][0];
        for (int k = threadIdx.x; k < kExpN; k += kTileThreads)
            sh.exptab[k] = make_double2(__longlong_as_double((long long)src[2 * k]),
                                        __longlong_as_double((long long)src[2 * k + 1]));
    }
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
    const float pxl = (float)lx + 0.5f, pyl = (float)ly + 0.5f;
    const double pxd = (double)px + 0.5, pyd = (double)py + 0.5;
    const uint32_t *__restrict__ gids = itp->gids;
    const Rec *__restrict__ recs = itp->recs;

    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
    bool done = !inside;
    float thr = log2_inv_eps() + 6e-5f;  // log2(T/EPS) + guard constant

    const int64_t s = itp->tstart[tl], e = itp->tend[tl];
    for (int64_t base = s; base < e; base += kTileThreads) {
        const int nb = (int)min((int64_t)kTileThreads, e - base);
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            const int t = threadIdx.x;
            const uint32_t gi = gids[base + t];
            const Rec r = recs[gi];
            const float mxl = (float)(r.mx - (double)ox), myl = (float)(r.my - (double)oy);
            sh.gid[t] = gi;
            sh.f0[t] = make_float4(mxl, myl, (float)(0.5 * kLog2e * r.ca), (float)(kLog2e * r.cb));
            sh.f1[t] = make_float2((float)(0.5 * kLog2e * r.cc), __log2f((float)r.al));
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
            if (USAGE) sh.cnt[t] = 0;
        }
        __syncthreads();
        for (int c = 0; c < nb; c += 32) {
            if (__all_sync(0xffffffffu, done)) break;
            const int jj = c + lane;
            unsigned m = __ballot_sync(0xffffffffu, jj < nb && ((sh.wmask[jj] >> w) & 1u));
            // phase A: fp32 candidate bits (T as of the chunk start; a larger T only
            // admits more candidates, never fewer)
            unsigned word = 0;
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                const float4 f0 = sh.f0[c + k];
                const float2 f1 = sh.f1[c + k];
                const float dx = pxl - f0.x, dy = pyl - f0.y;
                const float s2 = fmaf(f0.z * dx, dx, (f1.x * dy) * dy);  // log2e * 0.5(a dx^2 + c dy^2)
                const float e2 = fmaf(f0.w * dx, dy, s2);               // log2e * e
                // reject iff e > ln(al) + ln(T/EPS) + guard (guard proof: DESIGN.md)
                word |= (unsigned)(e2 <= fmaf(1e-5f, s2, f1.y) + thr) << k;
            }
            if (done) word = 0;
            // phase B: each lane runs its own candidates in depth order (exact fp64)
            while (word) {
                const int j1 = c + __ffs(word) - 1;
                word &= word - 1;
                const bool two = word != 0;
                const int j2 = two ? c + __ffs(word) - 1 : j1;
                word &= word - 1;
                const double ap1 = alpha_at(sh, j1, pxd, pyd);
                const double ap2 = alpha_at(sh, j2, pxd, pyd);
                double wgt = ap1 * T;
                if (wgt > kEpsContrib) {
                    const double2 rg = sh.rg[j1];
                    cr += wgt * rg.x;
                    cg += wgt * rg.y;
                    cb += wgt * sh.bl[j1];
                    T = T * (1.0 - ap1);
                    if (USAGE) atomicAdd(&sh.cnt[j1], 1);
                }
                if (two) {
                    wgt = ap2 * T;
                    if (wgt > kEpsContrib) {
                        const double2 rg = sh.rg[j2];
                        cr += wgt * rg.x;
                        cg += wgt * rg.y;
                        cb += wgt * sh.bl[j2];
                        T = T * (1.0 - ap2);
                        if (USAGE) atomicAdd(&sh.cnt[j2], 1);
                    }
                }
            }
            // once 0.999*T <= EPS no later primitive can pass the weight test
            done = done || kAlphaClamp * T <= kEpsContrib;
            thr = __log2f((float)T) + (log2_inv_eps() + 6e-5f);
        }
        __syncthreads();
        if (USAGE && (int)threadIdx.x < nb && sh.cnt[threadIdx.x] > 0)
            atomicAdd((unsigned long long *)(itp->usage + sh.gid[threadIdx.x]),
                      (unsigned long long)sh.cnt[threadIdx.x]);
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

// one block per item: fixed-order reduction of that item's tile partials
__global__ void __launch_bounds__(256)
k_sse_items(const double *__restrict__ sse_tiles, const int64_t *__restrict__ tile_base,
            const uint8_t *__restrict__ has_target, double *__restrict__ out) {
    const int s = blockIdx.x;
    if (!has_target[s]) return;
    const int64_t b = tile_base[s] * kCompWarps, n = (tile_base[s + 1] - tile_base[s]) * kCompWarps;
    double acc = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += 256) acc += sse_tiles[b + k];
    acc = warp_reduce_sum(acc);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        out[s] = t;
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
               uint32_t *__restrict__ vals) {
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
    int nt = 0;
    if (r.x1 > r.x0 && r.y1 > r.y0)
        nt = ((r.x1 - 1) / kTile - r.x0 / kTile + 1) * ((r.y1 - 1) / kTile - r.y0 / kTile + 1);
    ntiles[i] = nt;
    vals[i] = (uint32_t)i;
}

__global__ void k_fill_i64(int64_t *p, int64_t n, int64_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------
// host orchestration

struct ItemHost {
    int frame, cam;
    int64_t count;  // primitives of its frame
    int w, h, tiles_x, tiles_y;
    const double *target;
    double *image;
    double *trans;
    int64_t *usage;
    int clip;
};

// Stage B: given per item records (recs + item*stride), the depth-sorted
// primitive list vals (+ item*stride) of length nvis[item] (device), and
// ntiles per primitive, bin into tiles, composite and reduce SSE.
static void bin_and_composite(airgs_ctx *ctx, const std::vector<ItemHost> &items, int64_t stride,
                              const Rec *recs, const uint32_t *vals, const int32_t *ntiles,
                              const int64_t *d_nvis, int64_t max_nvis, double *sse, cudaStream_t st) {
    const int nitems = (int)items.size();
    int64_t &L = ctx->launches;
    // rank-ordered tile counts -> per-rank pair offsets, per-item totals
    int64_t *pair_off = ctx->scratch_t<int64_t>(kSlotPairOff, (size_t)nitems * stride);
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, (size_t)8 * nitems + 8);
    int64_t *d_npairs = stats + 4 * nitems;
    const int bps = (int)std::max<int64_t>(1, ceil_div(std::max<int64_t>(max_nvis, 1), kScanTile));
    int64_t *blocks = ctx->scratch_t<int64_t>(kSlotScanBlocks, (size_t)nitems * bps);
    if (max_nvis > 0) {
        seg_scan<int64_t>(TileCountIn{ntiles, vals, stride}, TileCountOut{pair_off, stride}, d_nvis, nitems,
                          max_nvis, blocks, d_npairs, st, &L);
    } else {
        AIRGS_CUDA_TRY(cudaMemsetAsync(d_npairs, 0, sizeof(int64_t) * nitems, st));
    }
    check_launch();
    std::vector<int64_t> npairs(nitems);
    AIRGS_CUDA_TRY(cudaMemcpyAsync(npairs.data(), d_npairs, sizeof(int64_t) * nitems, cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));

    // host layout: pair segments and tile bases
    std::vector<int64_t> hb(3 * nitems + 1);
    int64_t *pair_begin = hb.data();
    int64_t *tile_base = hb.data() + nitems;  // nitems + 1 entries
    int64_t P = 0, maxp = 0, Tt = 0;
    int max_tiles = 1;
    for (int s = 0; s < nitems; ++s) {
        pair_begin[s] = P;
        P += npairs[s];
        maxp = std::max(maxp, npairs[s]);
        tile_base[s] = Tt;
        Tt += (int64_t)items[s].tiles_x * items[s].tiles_y;
        max_tiles = std::max(max_tiles, items[s].tiles_x * items[s].tiles_y);
    }
    tile_base[nitems] = Tt;
    int64_t *d_pb = stats + 5 * nitems;  // pair_begin (nitems) then tile_base (nitems+1)
    AIRGS_CUDA_TRY(cudaMemcpyAsync(d_pb, hb.data(), sizeof(int64_t) * (2 * nitems + 1), cudaMemcpyHostToDevice, st));
    const int64_t *d_pair_begin = d_pb;
    const int64_t *d_tile_base = d_pb + nitems;

    uint32_t *pk = ctx->scratch_t<uint32_t>(kSlotPairKeys, (size_t)P);
    uint32_t *pv = ctx->scratch_t<uint32_t>(kSlotPairVals, (size_t)P);
    uint32_t *pk2 = ctx->scratch_t<uint32_t>(kSlotPairKeysAlt, (size_t)P);
    uint32_t *pv2 = ctx->scratch_t<uint32_t>(kSlotPairValsAlt, (size_t)P);
    int32_t *d_tiles_x = (int32_t *)ctx->scratch_t<int32_t>(kSlotMisc0, (size_t)nitems);
    {
        std::vector<int32_t> tx(nitems);
        for (int s = 0; s < nitems; ++s) tx[s] = items[s].tiles_x;
        AIRGS_CUDA_TRY(cudaMemcpyAsync(d_tiles_x, tx.data(), sizeof(int32_t) * nitems, cudaMemcpyHostToDevice, st));
        // tx is destroyed at scope end: make the copy complete first
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    if (P > 0 && max_nvis > 0) {
        EmitArgs ea{recs, vals, pair_off, d_nvis, d_pair_begin, d_tiles_x, pk, pv, stride};
        dim3 grid((unsigned)ceil_div(max_nvis, 256), (unsigned)nitems);
        k_emit_pairs<<<grid, 256, 0, st>>>(ea);
        ++L;
        check_launch();
        const int nbits = std::max(1, bit_length((uint64_t)(max_tiles - 1)));
        uint32_t *hist = ctx->scratch_t<uint32_t>(kSlotHist, (size_t)nitems * 256 * ceil_div(maxp, kSortTile));
        bool alt = radix_sort<uint32_t>(pk, pv, pk2, pv2, d_pair_begin, d_npairs, nitems, maxp, nbits, hist, st, &L);
        check_launch();
        if (alt) {
            std::swap(pk, pk2);
            std::swap(pv, pv2);
        }
    }
    int64_t *ranges = ctx->scratch_t<int64_t>(kSlotRanges, (size_t)2 * Tt);
    int64_t *tstart = ranges, *tend = ranges + Tt;
    AIRGS_CUDA_TRY(cudaMemsetAsync(ranges, 0, sizeof(int64_t) * 2 * Tt, st));
    if (P > 0) {
        dim3 grid((unsigned)ceil_div(maxp, 256), (unsigned)nitems);
        k_tile_ranges<<<grid, 256, 0, st>>>(pk, d_pair_begin, d_npairs, d_tile_base, tstart, tend);
        ++L;
        check_launch();
    }
    double *sse_tiles = ctx->scratch_t<double>(kSlotSseTiles, (size_t)Tt * kCompWarps);
    std::vector<CompItem> ci(nitems);
    std::vector<uint8_t> has_t(nitems);
    bool any_usage = false, any_target = false;
    for (int s = 0; s < nitems; ++s) {
        const ItemHost &h = items[s];
        CompItem &c = ci[s];
        c.recs = recs + (int64_t)s * stride;
        c.gids = pv + pair_begin[s];
        c.tstart = tstart + tile_base[s];
        c.tend = tend + tile_base[s];
        c.target = h.target;
        c.image = h.image;
        c.trans = h.trans;
        c.usage = h.usage;
        c.sse_tiles = sse_tiles + tile_base[s] * kCompWarps;
        c.w = h.w;
        c.h = h.h;
        c.tiles_x = h.tiles_x;
        c.clip = h.clip;
        any_usage |= h.usage != nullptr;
        any_target |= h.target != nullptr;
        has_t[s] = h.target != nullptr;
    }
    CompItem *d_ci = (CompItem *)ctx->scratch(kSlotMisc1, sizeof(CompItem) * nitems);
    uint8_t *d_has = (uint8_t *)ctx->scratch(kSlotMisc2, nitems);
    AIRGS_CUDA_TRY(cudaMemcpyAsync(d_ci, ci.data(), sizeof(CompItem) * nitems, cudaMemcpyHostToDevice, st));
    AIRGS_CUDA_TRY(cudaMemcpyAsync(d_has, has_t.data(), nitems, cudaMemcpyHostToDevice, st));
    if (Tt > 0) {
        if (any_usage)
            k_composite<true><<<(unsigned)Tt, kTileThreads, 0, st>>>(d_ci, d_tile_base, nitems);
        else
            k_composite<false><<<(unsigned)Tt, kTileThreads, 0, st>>>(d_ci, d_tile_base, nitems);
        ++L;
        check_launch();
    }
    if (sse && any_target) {
        k_sse_items<<<nitems, 256, 0, st>>>(sse_tiles, d_tile_base, d_has, sse);
        ++L;
        check_launch();
    }
    // host vectors (ci, has_t, hb) must outlive the async copies
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
}

static void render_impl(airgs_ctx *ctx, const airgs_frame *frames, int nframes, const airgs_camera *cams,
                        int ncams, const airgs_view_item *items, int nitems, double *sse, cudaStream_t st) {
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
        if (f.count > 0x7fffffffLL) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");
        const airgs_camera &c = cams[v.camera];
        if (c.width < 1 || c.height < 1) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad camera resolution");
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
        h.trans = nullptr;
        h.usage = v.usage;
        h.clip = 1;
        per_frame[v.frame].push_back(s);
        stride = std::max(stride, f.count);
    }
    int64_t &L = ctx->launches;
    // descriptors -> device (one packed upload)
    std::vector<int32_t> fptr(nframes + 1), fitems, icam(nitems);
    fptr[0] = 0;
    for (int f = 0; f < nframes; ++f) {
        for (int32_t s : per_frame[f]) fitems.push_back(s);
        fptr[f + 1] = (int32_t)fitems.size();
    }
    for (int s = 0; s < nitems; ++s) icam[s] = ih[s].cam;
    std::vector<int64_t> icount(nitems);
    for (int s = 0; s < nitems; ++s) icount[s] = ih[s].count;
    size_t off = 0;
    auto align = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t o_frames = off; off = align(off + sizeof(airgs_frame) * nframes);
    const size_t o_cams = off; off = align(off + sizeof(airgs_camera) * ncams);
    const size_t o_fptr = off; off = align(off + sizeof(int32_t) * (nframes + 1));
    const size_t o_fitems = off; off = align(off + sizeof(int32_t) * nitems);
    const size_t o_icam = off; off = align(off + sizeof(int32_t) * nitems);
    const size_t o_icount = off; off = align(off + sizeof(int64_t) * nitems);
    char *hs = (char *)ctx->staging(off);
    memcpy(hs + o_frames, frames, sizeof(airgs_frame) * nframes);
    memcpy(hs + o_cams, cams, sizeof(airgs_camera) * ncams);
    memcpy(hs + o_fptr, fptr.data(), sizeof(int32_t) * (nframes + 1));
    memcpy(hs + o_fitems, fitems.data(), sizeof(int32_t) * nitems);
    memcpy(hs + o_icam, icam.data(), sizeof(int32_t) * nitems);
    memcpy(hs + o_icount, icount.data(), sizeof(int64_t) * nitems);
    char *dd = (char *)ctx->scratch(kSlotDesc, off);
    AIRGS_CUDA_TRY(cudaMemcpyAsync(dd, hs, off, cudaMemcpyHostToDevice, st));

    // per-item stats: zmin, zmax, nvis, (npairs), ...
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, (size_t)8 * nitems + 8);
    unsigned long long *zmin = (unsigned long long *)stats;
    unsigned long long *zmax = (unsigned long long *)(stats + nitems);
    int64_t *nvis = stats + 2 * nitems;
    unsigned int *flags = ctx->scratch_t<unsigned int>(kSlotFlags, 4);
    {
        const int nb = (int)ceil_div(nitems, 256);
        k_fill_i64<<<nb, 256, 0, st>>>((int64_t *)zmin, nitems, -1);  // all ones
        k_fill_i64<<<nb, 256, 0, st>>>((int64_t *)zmax, 2 * nitems, 0);  // zmax + nvis
        L += 2;
        AIRGS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(unsigned int), st));
    }
    const size_t per = (size_t)nitems * stride;
    Rec *recs = ctx->scratch_t<Rec>(kSlotRecs, per);
    uint64_t *depth = ctx->scratch_t<uint64_t>(kSlotDepth, per);
    int32_t *ntiles = ctx->scratch_t<int32_t>(kSlotNtiles, per);
    uint64_t *keys = ctx->scratch_t<uint64_t>(kSlotKeys, per);
    uint32_t *vals = ctx->scratch_t<uint32_t>(kSlotVals, per);
    uint64_t *keys2 = ctx->scratch_t<uint64_t>(kSlotKeysAlt, per);
    uint32_t *vals2 = ctx->scratch_t<uint32_t>(kSlotValsAlt, per);

    ProjArgs pa;
    pa.frames = (const airgs_frame *)(dd + o_frames);
    pa.cams = (const airgs_camera *)(dd + o_cams);
    pa.frame_item_ptr = (const int32_t *)(dd + o_fptr);
    pa.frame_items = (const int32_t *)(dd + o_fitems);
    pa.item_cam = (const int32_t *)(dd + o_icam);
    pa.recs = recs;
    pa.depth = depth;
    pa.ntiles = ntiles;
    pa.zmin = zmin;
    pa.zmax = zmax;
    pa.flags = flags;
    pa.stride = stride;
    {
        dim3 grid((unsigned)ceil_div(stride, kProjThreads), (unsigned)nframes);
        k_project<<<grid, kProjThreads, 0, st>>>(pa);
        ++L;
        check_launch();
    }
    const int64_t *d_icount = (const int64_t *)(dd + o_icount);
    {
        const int bps = (int)std::max<int64_t>(1, ceil_div(stride, kScanTile));
        int64_t *blocks = ctx->scratch_t<int64_t>(kSlotScanBlocks, (size_t)nitems * bps);
        seg_scan<int64_t>(VisIn{ntiles, stride}, VisOut{depth, zmin, keys, vals, stride}, d_icount, nitems, stride,
                          blocks, nvis, st, &L);
        check_launch();
    }
    // readback: zmin, zmax, nvis, flags
    int64_t *hst = (int64_t *)ctx->staging(sizeof(int64_t) * (3 * nitems + 1));
    AIRGS_CUDA_TRY(cudaMemcpyAsync(hst, stats, sizeof(int64_t) * 3 * nitems, cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaMemcpyAsync(hst + 3 * nitems, flags, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned int hflags = *(unsigned int *)(hst + 3 * nitems);
    if (hflags & kFlagInvalidParam)
        throw ApiFailure(AIRGS_E_VALIDATION, "frame contains invalid primitive parameters");
    int64_t max_nvis = 0;
    uint64_t span = 0;
    for (int s = 0; s < nitems; ++s) {
        const int64_t nv = hst[2 * nitems + s];
        max_nvis = std::max(max_nvis, nv);
        if (nv > 0) span = std::max(span, (uint64_t)hst[nitems + s] - (uint64_t)hst[s]);
    }
    if (max_nvis > 0 && span > 0) {
        const int nbits = bit_length(span);
        uint32_t *hist = ctx->scratch_t<uint32_t>(kSlotHist, (size_t)nitems * 256 * ceil_div(max_nvis, kSortTile));
        // segment begins = s*stride: reuse a small device array
        int64_t *d_begin = ctx->scratch_t<int64_t>(kSlotMisc3, (size_t)nitems);
        std::vector<int64_t> hb(nitems);
        for (int s = 0; s < nitems; ++s) hb[s] = (int64_t)s * stride;
        AIRGS_CUDA_TRY(cudaMemcpyAsync(d_begin, hb.data(), sizeof(int64_t) * nitems, cudaMemcpyHostToDevice, st));
        bool alt = radix_sort<uint64_t>(keys, vals, keys2, vals2, d_begin, nvis, nitems, max_nvis, nbits, hist, st, &L);
        check_launch();
        if (alt) vals = vals2;
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));  // hb lifetime
    }
    bin_and_composite(ctx, ih, stride, recs, vals, ntiles, nvis, max_nvis, sse, st);
}

static void seam_impl(airgs_ctx *ctx, int64_t k, const double *means2d, const double *conics, const double *alphas,
                      const double *colors, const int64_t *bboxes, int h, int w, double *image, double *tfinal,
                      int64_t *usage, cudaStream_t st) {
    if (h < 1 || w < 1) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad image size");
    if (k > 0x7fffffffLL) throw ApiFailure(AIRGS_E_CAPACITY, "too many primitives");
    const int64_t stride = std::max<int64_t>(k, 1);
    Rec *recs = ctx->scratch_t<Rec>(kSlotRecs, stride);
    int32_t *ntiles = ctx->scratch_t<int32_t>(kSlotNtiles, stride);
    uint32_t *vals = ctx->scratch_t<uint32_t>(kSlotVals, stride);
    int64_t *stats = ctx->scratch_t<int64_t>(kSlotItemStats, 16);
    int64_t *nvis = stats + 2;
    if (usage && k > 0) AIRGS_CUDA_TRY(cudaMemsetAsync(usage, 0, sizeof(int64_t) * k, st));
    if (k > 0) {
        k_seam_records<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, means2d, conics, alphas, colors, bboxes, recs,
                                                                  ntiles, vals);
        ++ctx->launches;
        check_launch();
    }
    k_fill_i64<<<1, 32, 0, st>>>(nvis, 1, k);
    ++ctx->launches;
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
    // pixels never touched keep image 0 / T 1: the composite kernel writes
    // every in-image pixel of every tile, so no pre-fill is needed.
    bin_and_composite(ctx, ih, stride, recs, vals, ntiles, nvis, k, nullptr, st);
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

extern "C" int airgs_render(airgs_ctx *ctx, const airgs_frame *frames, int32_t nframes, const airgs_camera *cams,
                            int32_t ncams, const airgs_view_item *items, int32_t nitems, double *sse, void *stream) {
    return guarded(ctx, [&] { render_impl(ctx, frames, nframes, cams, ncams, items, nitems, sse, (cudaStream_t)stream); });
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

extern "C" int airgs_sse(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *out, void *stream) {
    return guarded(ctx, [&] { sse_impl(ctx, a, b, n, out, (cudaStream_t)stream); });
}
