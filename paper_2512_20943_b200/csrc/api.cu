// Context lifecycle of the airgs_b200 C-ABI.
#include <algorithm>
#include <cstring>

#include "context.h"

namespace airgs {

constexpr int kParamChunk = 3968;
struct ParamChunk {
    unsigned char b[kParamChunk];
};

__global__ void k_param_copy(unsigned char *__restrict__ dst, const ParamChunk c, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = c.b[i];
}

void h2d_small(airgs_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes > 16 * (size_t)kParamChunk) {
        // large block: DMA, and drain so the (reusable) host source may change afterwards
        AIRGS_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        AIRGS_CUDA_TRY(cudaStreamSynchronize(st));
        return;
    }
    const unsigned char *s = static_cast<const unsigned char *>(src);
    unsigned char *d = static_cast<unsigned char *>(dst);
    for (size_t off = 0; off < bytes; off += kParamChunk) {
        const int n = (int)std::min<size_t>(kParamChunk, bytes - off);
        ParamChunk c;
        memcpy(c.b, s + off, n);
        k_param_copy<<<1, 256, 0, st>>>(d + off, c, n);
        ++ctx->launches;
    }
    check_launch();
}

}  // namespace airgs

using namespace airgs;

extern "C" int airgs_ctx_create(airgs_ctx **out, int32_t device) {
    if (!out) return AIRGS_E_INTERNAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return AIRGS_E_CUDA;
    if (cudaSetDevice(device) != cudaSuccess) return AIRGS_E_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return AIRGS_E_CUDA;
    if (prop.major < 10) return AIRGS_E_CUDA;  // built for sm_100a only
    airgs_ctx *c = new (std::nothrow) airgs_ctx();
    if (!c) return AIRGS_E_INTERNAL;
    c->device = device;
    *out = c;
    return AIRGS_OK;
}

extern "C" int airgs_ctx_destroy(airgs_ctx *ctx) {
    if (!ctx) return AIRGS_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->d_stats) cudaFree(ctx->d_stats);
    if (ctx->d_defer) cudaFree(ctx->d_defer);
    delete ctx;
    return AIRGS_OK;
}

extern "C" const char *airgs_last_error(const airgs_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

extern "C" int64_t airgs_launch_count(const airgs_ctx *ctx) { return ctx ? ctx->launches : 0; }

extern "C" int airgs_timing(airgs_ctx *ctx, int32_t enable, double *composite_ms, int64_t *composite_launches,
                            double *project_ms, int64_t *project_launches) {
    double ms[airgs_ctx::kStages];
    int64_t n[airgs_ctx::kStages];
    const int rc = airgs_timing_stages(ctx, enable, ms, n, airgs_ctx::kStages);
    if (rc) return rc;
    if (composite_ms) *composite_ms = ms[kStageComposite];
    if (composite_launches) *composite_launches = n[kStageComposite];
    if (project_ms) *project_ms = ms[kStageProject];
    if (project_launches) *project_launches = n[kStageProject];
    return AIRGS_OK;
}

extern "C" int airgs_timing_stages(airgs_ctx *ctx, int32_t enable, double *ms, int64_t *launches, int32_t nstages) {
    if (!ctx) return AIRGS_E_INTERNAL;
    try {
        cudaSetDevice(ctx->device);
        ctx->resolve_timing();
    } catch (...) {
        return AIRGS_E_CUDA;
    }
    for (int k = 0; k < nstages; ++k) {
        const bool in = k < airgs_ctx::kStages;
        if (ms) ms[k] = in ? ctx->stage_ms[k] : 0.0;
        if (launches) launches[k] = in ? ctx->stage_launches[k] : 0;
    }
    if (enable >= 0) {  // (re)arm or disarm and reset the counters
        ctx->timing = enable != 0;
        for (int k = 0; k < airgs_ctx::kStages; ++k) {
            ctx->stage_ms[k] = 0.0;
            ctx->stage_launches[k] = 0;
        }
    }
    return AIRGS_OK;
}

static int stats_reset(airgs_ctx *ctx) {
    unsigned long long h[airgs::kStatSlots];
    for (int k = 0; k < airgs::kStatSlots; ++k) h[k] = 0ull;
    const unsigned long long inf = 0x7ff0000000000000ull;  // +inf bits: min slots start empty
    h[airgs::kMarginWeight] = h[airgs::kMarginTerm] = h[airgs::kMarginDepthGap] = inf;
    h[airgs::kMarginBBox] = h[airgs::kMarginNear] = h[airgs::kMarginAlpha] = inf;
    return cudaMemcpy(ctx->d_stats, h, sizeof(h), cudaMemcpyHostToDevice) == cudaSuccess ? AIRGS_OK : AIRGS_E_CUDA;
}

static int stats_read(airgs_ctx *ctx, unsigned long long *h) {
    for (int k = 0; k < airgs::kStatSlots; ++k) h[k] = 0ull;
    if (!ctx->d_stats) return AIRGS_OK;
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(h, ctx->d_stats, sizeof(unsigned long long) * airgs::kStatSlots, cudaMemcpyDeviceToHost) !=
            cudaSuccess) {
        ctx->err = "eval stats readback failed";
        return AIRGS_E_CUDA;
    }
    return AIRGS_OK;
}

extern "C" int airgs_eval_stats(airgs_ctx *ctx, int32_t enable, int64_t *counts) {
    if (!ctx) return AIRGS_E_INTERNAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return AIRGS_E_CUDA;
    unsigned long long h[airgs::kStatSlots];
    if (int rc = stats_read(ctx, h)) return rc;
    if (counts)
        for (int k = 0; k < 3; ++k) counts[k] = (int64_t)h[k];
    if (counts) {
        counts[3] = (int64_t)h[airgs::kStatTilePairs];
        counts[4] = (int64_t)h[airgs::kStatRecords];
    }
    if (enable >= 0) {  // (re)arm or disarm and reset the counters
        if (enable && !ctx->d_stats &&
            cudaMalloc(&ctx->d_stats, sizeof(unsigned long long) * airgs::kStatSlots) != cudaSuccess) {
            ctx->err = "eval stats allocation failed";
            return AIRGS_E_CUDA;
        }
        if (ctx->d_stats)
            if (int rc = stats_reset(ctx)) return rc;
        ctx->stats = enable != 0;
    }
    return AIRGS_OK;
}

extern "C" int airgs_defer(airgs_ctx *ctx, int32_t enable, uint32_t *flags_out) {
    if (!ctx) return AIRGS_E_INTERNAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return AIRGS_E_CUDA;
    if (enable) {
        if (!ctx->d_defer && cudaMalloc(&ctx->d_defer, sizeof(unsigned int)) != cudaSuccess) return AIRGS_E_CUDA;
        if (cudaMemset(ctx->d_defer, 0, sizeof(unsigned int)) != cudaSuccess) return AIRGS_E_CUDA;
        ctx->defer = true;
        if (flags_out) *flags_out = 0;
        return AIRGS_OK;
    }
    unsigned int h = 0;
    if (ctx->d_defer) {
        if (cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(&h, ctx->d_defer, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
            return AIRGS_E_CUDA;
    }
    ctx->defer = false;
    if (flags_out) *flags_out = h;
    return AIRGS_OK;
}

extern "C" int airgs_eval_margins(airgs_ctx *ctx, double *margins) {
    if (!ctx || !margins) return AIRGS_E_INTERNAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return AIRGS_E_CUDA;
    unsigned long long h[airgs::kStatSlots];
    if (int rc = stats_read(ctx, h)) return rc;
    for (int k = 0; k < 7; ++k) {
        const int slot = airgs::kMarginWeight + k;
        double v;
        std::memcpy(&v, &h[slot], sizeof(v));
        margins[k] = slot == airgs::kMarginDepthTies ? (double)h[slot] : v;
    }
    return AIRGS_OK;
}
