// Windowed SSIM and its gradient, L1 and its gradient (ss/metrics.py:47-121),
// the image terms of the reference trainer's loss (ss/train.py:110-114).
//
// SSIM (ss/metrics.py:62-86): luminance = channel mean ((r + g) + b) / 3,
// five valid-mode 11x11 Gaussian-window moments (mu_a, mu_b, E[a^2], E[b^2],
// E[ab]), per-window a1 a2 / (b1 b2), mean over the valid windows.  The
// window is separable (outer(g, g) / sum = outer(g/sum g, g/sum g)), so each
// moment is a horizontal then a vertical 11-tap pass (22 instead of 121
// multiply-adds per output); the result agrees with scipy's direct 2D sum to
// rounding (~1e-16 relative), not bit for bit -- scipy's summation order is
// not a fixed loop order (checked here against every simple order).
//
// Gradient (ss/metrics.py:89-113): the three per-window adjoints d_mu_a,
// d_t_a, d_t_ab, full-mode convolved with the window (again separable), then
// g = conv(d_mu_a) + 2 la conv(d_t_a) + lb conv(d_t_ab), / n_windows, / 3 per
// channel for colour images.
//
// All passes are HBM/L2 streaming stencils over fp64 maps; reductions are
// fixed-order (deterministic).
#include "context.h"
#include "scan_sort.cuh"

namespace airgs {

constexpr int kWin = 11;  // window edge (radius 5)
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;

struct Win {
    double g[kWin];  // normalised 1-D window (host-computed as the reference's g / sum g)
};

__device__ __forceinline__ double lum(const double *__restrict__ p, int64_t pix, int ch) {
    if (ch == 1) return p[pix];
    const double *q = p + 3 * pix;
    return ((q[0] + q[1]) + q[2]) / 3.0;  // numpy mean over 3 channels
}

// horizontal valid pass of the five moment images: H[m][y][x], x in [0, ow)
__global__ void __launch_bounds__(256) k_ssim_h(const double *__restrict__ a, const double *__restrict__ b, int h,
                                                int w, int ch, Win win, double *__restrict__ H) {
    const int ow = w - kWin + 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)h * ow) return;
    const int y = (int)(i / ow), x = (int)(i % ow);
    double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const int64_t pix = (int64_t)y * w + x + k;
        const double la = lum(a, pix, ch), lb = lum(b, pix, ch), gk = win.g[k];
        s[0] += gk * la;
        s[1] += gk * lb;
        s[2] += gk * (la * la);
        s[3] += gk * (lb * lb);
        s[4] += gk * (la * lb);
    }
    const int64_t plane = (int64_t)h * ow;
#pragma unroll
    for (int m = 0; m < 5; ++m) H[m * plane + i] = s[m];
}

// vertical valid pass + per-window SSIM terms; per-block partial sums of the
// SSIM map (fixed order) and, for the gradient, the three adjoint maps
__global__ void __launch_bounds__(256) k_ssim_v(const double *__restrict__ H, int h, int w, Win win,
                                                double *__restrict__ part, double *__restrict__ D) {
    const int ow = w - kWin + 1, oh = h - kWin + 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sv = 0.0;
    if (i < (int64_t)oh * ow) {
        const int y = (int)(i / ow), x = (int)(i % ow);
        const int64_t plane = (int64_t)h * ow;
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            const int64_t r = (int64_t)(y + j) * ow + x;
            const double gj = win.g[j];
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] += gj * H[q * plane + r];
        }
        const double mu_a = m[0], mu_b = m[1], t_a = m[2], t_b = m[3], t_ab = m[4];
        // ss/metrics.py:68-72
        const double a1 = 2.0 * mu_a * mu_b + kC1;
        const double a2 = 2.0 * (t_ab - mu_a * mu_b) + kC2;
        const double b1 = mu_a * mu_a + mu_b * mu_b + kC1;
        const double b2 = (t_a - mu_a * mu_a) + (t_b - mu_b * mu_b) + kC2;
        const double denom = b1 * b2;
        sv = a1 * a2 / denom;
        if (D) {  // ss/metrics.py:99-101
            const int64_t op = (int64_t)oh * ow;
            D[i] = (2.0 * mu_b * a2 - 2.0 * mu_b * a1) / denom - sv * (2.0 * mu_a / b1 - 2.0 * mu_a / b2);
            D[op + i] = -sv / b2;
            D[2 * op + i] = 2.0 * a1 / denom;
        }
    }
    sv = warp_reduce_sum(sv);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sv;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

// fixed-order sum of n partials (one block)
__global__ void __launch_bounds__(256) k_sum_parts(const double *__restrict__ part, int64_t n, double count,
                                                   double *__restrict__ out) {
    double acc = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += 256) acc += part[k];
    acc = warp_reduce_sum(acc);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        *out = t / count;
    }
}

// horizontal full pass of the three adjoint maps: F[m][y][x], y in [0, oh), x in [0, w)
__global__ void __launch_bounds__(256) k_ssim_full_h(const double *__restrict__ D, int h, int w, Win win,
                                                     double *__restrict__ F) {
    const int ow = w - kWin + 1, oh = h - kWin + 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)oh * w) return;
    const int y = (int)(i / w), x = (int)(i % w);
    const int64_t op = (int64_t)oh * ow, fp = (int64_t)oh * w;
    double s[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const int xs = x - k;
        if (xs < 0 || xs >= ow) continue;
        const double gk = win.g[k];
        const int64_t r = (int64_t)y * ow + xs;
#pragma unroll
        for (int q = 0; q < 3; ++q) s[q] += gk * D[q * op + r];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) F[q * fp + i] = s[q];
}

// vertical full pass + combination: grad (h, w, ch)
__global__ void __launch_bounds__(256) k_ssim_full_v(const double *__restrict__ F, const double *__restrict__ a,
                                                     const double *__restrict__ b, int h, int w, int ch, Win win,
                                                     double nwin, double *__restrict__ grad) {
    const int oh = h - kWin + 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)h * w) return;
    const int y = (int)(i / w), x = (int)(i % w);
    const int64_t fp = (int64_t)oh * w;
    double s[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
        const int ys = y - j;
        if (ys < 0 || ys >= oh) continue;
        const double gj = win.g[j];
        const int64_t r = (int64_t)ys * w + x;
#pragma unroll
        for (int q = 0; q < 3; ++q) s[q] += gj * F[q * fp + r];
    }
    const double la = lum(a, i, ch), lb = lum(b, i, ch);
    const double g = ((s[0] + 2.0 * la * s[1]) + lb * s[2]) / nwin;
    if (ch == 1) {
        grad[i] = g;
    } else {
        const double g3 = g / 3.0;
        grad[3 * i] = g3;
        grad[3 * i + 1] = g3;
        grad[3 * i + 2] = g3;
    }
}

// L1: per-block partial sums of |a - b|; optional gradient sign(a - b) / n
__global__ void __launch_bounds__(256) k_l1(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                                            double inv_n, double *__restrict__ part, double *__restrict__ grad) {
    double acc = 0.0;
    const int64_t per = ceil_div(n, (int64_t)gridDim.x);
    const int64_t lo = per * blockIdx.x, hi = min(n, lo + per);
    for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
        const double d = a[i] - b[i];
        acc += fabs(d);
        if (grad) grad[i] = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;
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

static void ssim_impl(airgs_ctx *ctx, const double *a, const double *b, int h, int w, int ch, const double *win,
                      double *ssim_out, double *grad, cudaStream_t st) {
    if (ch != 1 && ch != 3) throw ApiFailure(AIRGS_E_STRUCTURAL, "images must be (h, w) or (h, w, 3)");
    if (h < kWin || w < kWin) throw ApiFailure(AIRGS_E_STRUCTURAL, "image smaller than the 11x11 SSIM window");
    Win wn;
    for (int k = 0; k < kWin; ++k) wn.g[k] = win[k];
    const int ow = w - kWin + 1, oh = h - kWin + 1;
    const int64_t nh = (int64_t)h * ow, nv = (int64_t)oh * ow;
    double *H = ctx->scratch_t<double>(kSlotMetric0, (size_t)5 * nh);
    const unsigned gv = (unsigned)ceil_div(nv, (int64_t)256);
    double *part = ctx->scratch_t<double>(kSlotMetric1, gv);
    double *D = grad ? ctx->scratch_t<double>(kSlotMetric2, (size_t)3 * nv) : nullptr;
    k_ssim_h<<<(unsigned)ceil_div(nh, (int64_t)256), 256, 0, st>>>(a, b, h, w, ch, wn, H);
    k_ssim_v<<<gv, 256, 0, st>>>(H, h, w, wn, part, D);
    k_sum_parts<<<1, 256, 0, st>>>(part, gv, (double)nv, ssim_out);
    ctx->launches += 3;
    check_launch();
    if (grad) {
        const int64_t nf = (int64_t)oh * w;
        double *F = ctx->scratch_t<double>(kSlotMetric0, (size_t)std::max<int64_t>(3 * nf, 5 * nh));
        k_ssim_full_h<<<(unsigned)ceil_div(nf, (int64_t)256), 256, 0, st>>>(D, h, w, wn, F);
        k_ssim_full_v<<<(unsigned)ceil_div((int64_t)h * w, (int64_t)256), 256, 0, st>>>(F, a, b, h, w, ch, wn,
                                                                                       (double)nv, grad);
        ctx->launches += 2;
        check_launch();
    }
}

static void l1_impl(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *l1_out, double *grad,
                    cudaStream_t st) {
    if (n <= 0) throw ApiFailure(AIRGS_E_STRUCTURAL, "empty images");
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(1184, ceil_div(n, (int64_t)4096)));
    double *part = ctx->scratch_t<double>(kSlotMetric1, parts);
    k_l1<<<parts, 256, 0, st>>>(a, b, n, 1.0 / (double)n, part, grad);
    k_sum_parts<<<1, 256, 0, st>>>(part, parts, (double)n, l1_out);
    ctx->launches += 2;
    check_launch();
}

}  // namespace airgs

using namespace airgs;

extern "C" int airgs_ssim(airgs_ctx *ctx, const double *a, const double *b, int32_t height, int32_t width,
                          int32_t channels, const double *window, double *ssim_out, double *grad, void *stream) {
    return guarded(ctx, [&] { ssim_impl(ctx, a, b, height, width, channels, window, ssim_out, grad, (cudaStream_t)stream); });
}

extern "C" int airgs_l1(airgs_ctx *ctx, const double *a, const double *b, int64_t n, double *l1_out, double *grad,
                        void *stream) {
    return guarded(ctx, [&] { l1_impl(ctx, a, b, n, l1_out, grad, (cudaStream_t)stream); });
}
