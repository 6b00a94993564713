// Shared definitions for the airgs_b200 CUDA library (sm_100a).
//
// The whole library is compiled with -fmad=false: every a*b+c in this code
// is a separate multiply and add, exactly like numpy's elementwise ops and
// the reference's Cython kernel.  Where the reference goes through OpenBLAS
// (which fuses) we call fma() explicitly; where we want FMA for speed in the
// fp32 fast-reject path we call fmaf()/__fmaf_rn explicitly.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "../../include/airgs_b200.h"

namespace airgs {

constexpr int kTile = 16;            // screen tile edge (pixels)
constexpr int kTileThreads = 256;    // one thread per tile pixel
constexpr double kEpsContrib = 1.0 / 255.0;  // _composite.pyx:14
constexpr double kAlphaClamp = 0.999;        // _composite.pyx:15
constexpr double kCovBlur = 0.3;             // rasterizer.py:52
constexpr double kRadiusSigma = 3.5;         // rasterizer.py:53
constexpr double kShC0 = 0.2820947917738781; // rasterizer.py:55
constexpr double kShC1 = 0.4886025119029199; // rasterizer.py:56

// Per (view item, primitive) projected record -- everything the exact fp64
// compositing path needs, 96 bytes, 16-byte aligned for vector loads.
struct __align__(16) Rec {
    double mx, my;        // projected mean (pixels)
    double ca, cb, cc;    // conic (a, b, c) = (c2, -b2, a2) / det
    double al;            // activated opacity
    double cr, cg, cbl;   // activated colour
    int32_t x0, x1, y0, y1;  // clipped bbox [x0,x1) x [y0,y1)
    // half extents of the AABB of the ellipse e <= ln(al/EPS) (+ outward pad):
    // no pixel centre outside it can pass the weight test
    float hx, hy;
};
static_assert(sizeof(Rec) == 96, "Rec layout");

struct Status {
    int code = AIRGS_OK;
    std::string msg;
};

// device-side error flags (bitmask) written by kernels
// Diagnostic decision margins (airgs_eval_margins): non-negative doubles kept
// as their bit patterns (integer order = value order), min-reduced per warp
// then one atomicMin per warp.
enum MarginSlot {
    kMarginWeight = 3,       // min |w - 1/255| / (1/255) over every weight test
    kMarginTerm = 4,         // min |0.999 T - 1/255| / (1/255) after every contribution
    kMarginDepthGap = 5,     // min gap (ulps) between adjacent distinct depth keys of a tile list
    kMarginDepthTies = 6,    // adjacent equal depth keys (resolved by index)
    kMarginBBox = 7,         // min distance of a bbox floor/ceil argument to an integer (px)
    kMarginNear = 8,         // min |z - near_clip|
    kMarginAlpha = 9,        // min |alpha - 1/255| / (1/255) (opacity cull)
    kStatTilePairs = 10,     // (tile, primitive) list entries after binning (counter)
    kStatRecords = 11,       // projected records written (primitives reaching >= 1 tile, per view)
    kStatSlots = 12
};

enum DevFlag : unsigned int {
    kFlagInvalidParam = 1u,   // zero quaternion / non-finite parameter
    kFlagDecodeTrunc = 2u,    // varint section inconsistent
    kFlagVarintLong = 4u,     // varint longer than 10 bytes
    kFlagIndexRange = 8u,     // delta index >= base_count
    kFlagQuantOverflow = 16u, // |q| > 2^31-1
    kFlagBucketOverflow = 32u, // a tile received more primitives than its bucket holds
    kDeferDecode = 64u,        // deferred mode: a GSDP decode failed its checks
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int bit_length(uint64_t v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b;
}

}  // namespace airgs

#define AIRGS_CUDA_TRY(expr)                                                         \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            throw ::airgs::CudaFailure(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
        }                                                                            \
    } while (0)

namespace airgs {
struct CudaFailure {
    std::string what;
    explicit CudaFailure(std::string w) : what(std::move(w)) {}
};
struct ApiFailure {
    int code;
    std::string what;
    ApiFailure(int c, std::string w) : code(c), what(std::move(w)) {}
};
}  // namespace airgs
