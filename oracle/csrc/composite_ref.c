/*
 * CPU ORACLE -- test infrastructure only.  Nothing in the product path links
 * or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it (as the checker or the timed
 * CPU arm).
 *
 * Restatement of the reference compositing loop
 *   /root/reference/pkg/src/splatstream/_composite.pyx:18-74  (forward)
 * in plain C, compiled with -ffp-contract=off so that every `x*y + z` is a
 * separate multiply and add, exactly like the Cython-generated C
 * (numerics contract).
 *
 * Two iteration orders are provided:
 *   oracle_composite_gmajor  -- Gaussian-major over each clipped bbox, the
 *                               reference's own order (no early exit);
 *   oracle_composite_tiles   -- pixel-major over 16x16 tile candidate lists
 *                               in depth order with exact early termination
 *                               (0.999*T <= 1/255).  This is the iteration
 *                               order of the CUDA kernel; the two must agree
 *                               bit-for-bit (SURVEY.md s7 hard part 3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const double K_EPS = 1.0 / 255.0;   /* _composite.pyx:14 */
static const double K_CLAMP = 0.999;       /* _composite.pyx:15 */

void oracle_composite_gmajor(int64_t k, const double *means2d, const double *conics,
                             const double *alphas, const double *colors,
                             const int64_t *bboxes, int height, int width,
                             double *image, double *trans, int64_t *usage)
{
    int64_t npx = (int64_t)height * width;
    for (int64_t p = 0; p < npx; ++p) {
        image[3 * p] = image[3 * p + 1] = image[3 * p + 2] = 0.0;
        trans[p] = 1.0;
    }
    for (int64_t i = 0; i < k; ++i) {
        int x0 = (int)bboxes[4 * i], x1 = (int)bboxes[4 * i + 1];
        int y0 = (int)bboxes[4 * i + 2], y1 = (int)bboxes[4 * i + 3];
        usage[i] = 0;
        if (x1 <= x0 || y1 <= y0) continue;
        double mx = means2d[2 * i], my = means2d[2 * i + 1];
        double a = conics[3 * i], b = conics[3 * i + 1], c = conics[3 * i + 2];
        double al = alphas[i];
        double cr = colors[3 * i], cg = colors[3 * i + 1], cb = colors[3 * i + 2];
        int64_t cnt = 0;
        for (int iy = y0; iy < y1; ++iy) {
            double dy = ((double)iy + 0.5) - my;
            for (int ix = x0; ix < x1; ++ix) {
                double dx = ((double)ix + 0.5) - mx;
                double e = 0.5 * (a * dx * dx + c * dy * dy) + b * dx * dy;
                double ap = al * exp(-e);
                if (ap > K_CLAMP) ap = K_CLAMP;
                int64_t p = (int64_t)iy * width + ix;
                double t = trans[p];
                double w = ap * t;
                if (w > K_EPS) {
                    image[3 * p] += w * cr;
                    image[3 * p + 1] += w * cg;
                    image[3 * p + 2] += w * cb;
                    trans[p] = t * (1.0 - ap);
                    ++cnt;
                }
            }
        }
        usage[i] = cnt;
    }
}

/* Pixel-major restatement.  Tile candidate lists hold primitive positions in
 * depth order (the input order), built from the same clipped bboxes.  A pixel
 * stops once 0.999*T <= 1/255: from then on w = min(al*g,0.999)*T rounds to a
 * value <= 1/255 for every later primitive, so stopping is exact. */
void oracle_composite_tiles(int64_t k, const double *means2d, const double *conics,
                            const double *alphas, const double *colors,
                            const int64_t *bboxes, int height, int width, int tile,
                            double *image, double *trans, int64_t *usage)
{
    int tx = (width + tile - 1) / tile, ty = (height + tile - 1) / tile;
    int64_t ntiles = (int64_t)tx * ty;
    int64_t *cnt = (int64_t *)calloc((size_t)ntiles + 1, sizeof(int64_t));
    for (int64_t i = 0; i < k; ++i) {
        usage[i] = 0;
        int64_t x0 = bboxes[4 * i], x1 = bboxes[4 * i + 1], y0 = bboxes[4 * i + 2], y1 = bboxes[4 * i + 3];
        if (x1 <= x0 || y1 <= y0) continue;
        for (int64_t v = y0 / tile; v <= (y1 - 1) / tile; ++v)
            for (int64_t u = x0 / tile; u <= (x1 - 1) / tile; ++u) cnt[v * tx + u + 1]++;
    }
    for (int64_t t = 0; t < ntiles; ++t) cnt[t + 1] += cnt[t];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntiles + 1));
    memcpy(fill, cnt, sizeof(int64_t) * (size_t)(ntiles + 1));
    int64_t *list = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt[ntiles] + 1));
    for (int64_t i = 0; i < k; ++i) {
        int64_t x0 = bboxes[4 * i], x1 = bboxes[4 * i + 1], y0 = bboxes[4 * i + 2], y1 = bboxes[4 * i + 3];
        if (x1 <= x0 || y1 <= y0) continue;
        for (int64_t v = y0 / tile; v <= (y1 - 1) / tile; ++v)
            for (int64_t u = x0 / tile; u <= (x1 - 1) / tile; ++u) list[fill[v * tx + u]++] = i;
    }
    for (int v = 0; v < ty; ++v)
        for (int u = 0; u < tx; ++u) {
            int64_t t = (int64_t)v * tx + u;
            for (int iy = v * tile; iy < (v + 1) * tile && iy < height; ++iy)
                for (int ix = u * tile; ix < (u + 1) * tile && ix < width; ++ix) {
                    double r = 0.0, g = 0.0, bl = 0.0, T = 1.0;
                    for (int64_t j = cnt[t]; j < cnt[t + 1]; ++j) {
                        if (K_CLAMP * T <= K_EPS) break;
                        int64_t i = list[j];
                        double dx = ((double)ix + 0.5) - means2d[2 * i];
                        double dy = ((double)iy + 0.5) - means2d[2 * i + 1];
                        double a = conics[3 * i], b = conics[3 * i + 1], c = conics[3 * i + 2];
                        double e = 0.5 * (a * dx * dx + c * dy * dy) + b * dx * dy;
                        double ap = alphas[i] * exp(-e);
                        if (ap > K_CLAMP) ap = K_CLAMP;
                        double w = ap * T;
                        if (w > K_EPS) {
                            r += w * colors[3 * i];
                            g += w * colors[3 * i + 1];
                            bl += w * colors[3 * i + 2];
                            T = T * (1.0 - ap);
                            usage[i]++;
                        }
                    }
                    int64_t p = (int64_t)iy * width + ix;
                    image[3 * p] = r;
                    image[3 * p + 1] = g;
                    image[3 * p + 2] = bl;
                    trans[p] = T;
                }
        }
    free(list);
    free(fill);
    free(cnt);
}

/* Correctly rounded fused multiply-add, used by the numpy restatement to
 * mirror OpenBLAS' FMA accumulation order in the projection matmuls
 * (ss/rasterizer.py:119,159,166-167). */
void oracle_fma(int64_t n, const double *a, const double *b, const double *c, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
}

/* Evaluation counts of the reference loop:
 * counts[0] = (pixel, primitive) pairs inside clipped bboxes, counts[1] =
 * those whose pixel was still live (0.999*T > 1/255 before the evaluation),
 * counts[2] = contributing pairs.  Same arithmetic as the gmajor loop. */
void oracle_eval_counts(int64_t k, const double *means2d, const double *conics,
                        const double *alphas, const double *bboxes_unused, const int64_t *bboxes,
                        int height, int width, int64_t *counts)
{
    (void)bboxes_unused;
    int64_t npx = (int64_t)height * width;
    double *trans = (double *)malloc(sizeof(double) * (size_t)(npx > 0 ? npx : 1));
    for (int64_t p = 0; p < npx; ++p) trans[p] = 1.0;
    counts[0] = counts[1] = counts[2] = 0;
    for (int64_t i = 0; i < k; ++i) {
        int x0 = (int)bboxes[4 * i], x1 = (int)bboxes[4 * i + 1];
        int y0 = (int)bboxes[4 * i + 2], y1 = (int)bboxes[4 * i + 3];
        if (x1 <= x0 || y1 <= y0) continue;
        double mx = means2d[2 * i], my = means2d[2 * i + 1];
        double a = conics[3 * i], b = conics[3 * i + 1], c = conics[3 * i + 2];
        double al = alphas[i];
        for (int iy = y0; iy < y1; ++iy) {
            double dy = ((double)iy + 0.5) - my;
            for (int ix = x0; ix < x1; ++ix) {
                int64_t p = (int64_t)iy * width + ix;
                double t = trans[p];
                counts[0] += 1;
                if (K_CLAMP * t > K_EPS) counts[1] += 1;
                double dx = ((double)ix + 0.5) - mx;
                double e = 0.5 * (a * dx * dx + c * dy * dy) + b * dx * dy;
                double ap = al * exp(-e);
                if (ap > K_CLAMP) ap = K_CLAMP;
                if (ap * t > K_EPS) {
                    trans[p] = t * (1.0 - ap);
                    counts[2] += 1;
                }
            }
        }
    }
    free(trans);
}
