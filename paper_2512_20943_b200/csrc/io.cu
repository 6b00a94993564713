// Parameter transfer layout: row-major little-endian float64 rows (the
// reference's GaussianFrame.params and the GSSC scene container's payload,
// ss/model.py:318-350) -> the plane-major device layout of every kernel.
// The source may start at any byte offset (GSSC rows start at byte 15 of the
// file), so unaligned sources are assembled from bytes.
#include "context.h"

namespace airgs {

__global__ void __launch_bounds__(256) k_rows_to_planes_aligned(const double *__restrict__ src, int64_t n, int W,
                                                                double *__restrict__ planes, int64_t ld) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n * W) return;
    const int64_t i = k / W;
    const int c = (int)(k - i * W);
    planes[(int64_t)c * ld + i] = src[k];
}

__global__ void __launch_bounds__(256) k_rows_to_planes_bytes(const uint8_t *__restrict__ src, int64_t n, int W,
                                                              double *__restrict__ planes, int64_t ld) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n * W) return;
    const uint8_t *p = src + 8 * k;
    unsigned long long v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) v |= (unsigned long long)p[b] << (8 * b);
    const int64_t i = k / W;
    const int c = (int)(k - i * W);
    planes[(int64_t)c * ld + i] = __longlong_as_double((long long)v);
}

}  // namespace airgs

using namespace airgs;

extern "C" int airgs_rows_to_planes(airgs_ctx *ctx, const uint8_t *bytes, int64_t byte_offset, int64_t n,
                                    int32_t width, double *planes, int64_t ld, void *stream) {
    return guarded(ctx, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        if (n < 0 || width <= 0 || ld < n) throw ApiFailure(AIRGS_E_STRUCTURAL, "bad parameter layout");
        if (n == 0) return;
        const uint8_t *src = bytes + byte_offset;
        const unsigned grid = (unsigned)ceil_div(n * (int64_t)width, (int64_t)256);
        if (((uintptr_t)src & 7u) == 0)
            k_rows_to_planes_aligned<<<grid, 256, 0, st>>>(reinterpret_cast<const double *>(src), n, width, planes, ld);
        else
            k_rows_to_planes_bytes<<<grid, 256, 0, st>>>(src, n, width, planes, ld);
        ++ctx->launches;
        check_launch();
    });
}
