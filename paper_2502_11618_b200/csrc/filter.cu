// Hierarchical depth filter (filtering.py:60-147) + frame assembly
// (render.py:146-161) + U-Net input packing (weights.ts:90-95, bridge.ts:37-44).
//
// Per frame (fast path) this is L+1 launches:
//   k_assemble_pyramid  one CTA per 32x32 pixel block: integer-mean colours,
//                       f32 depth/alpha, sentinel conversion and up to five 2x2
//                       min-pool levels in shared memory; consumes and resets the
//                       projection buffers for the next frame.
//   k_filter_step<F>    one thread per COARSE pixel: Laplacian edge + reference
//                       depth of the parent (3x3 window), keep test of its <= 4
//                       children, renormalised bilinear fill (non-final steps).
//                       The final step applies the mask to the frame and writes
//                       the U-Net input.
// Each output pixel depends only on a 3x3 coarse window, so every step is a
// pure stencil; the working set (<= 8 MB at 1080p) stays in L2.
#include <atomic>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "ls_common.cuh"

namespace ls {

__device__ __forceinline__ float sentinel(float d) { return d <= 0.0f ? INFINITY : d; }

// The stencil helpers read the image through an accessor get(y, x) (only ever
// called for in-image coordinates), so the global-memory kernels and the
// fused shared-memory steps run the same arithmetic.

// _native.pyx:173-196 at one pixel
template <typename Get>
__device__ __forceinline__ bool lap_edge_t(Get get, int64_t h, int64_t w, int64_t y, int64_t x,
                                           double thr) {
    const double c = (double)get(y, x);
    if (!finite_d(c)) return false;
    double up = y > 0 ? (double)get(y - 1, x) : c;
    double dn = y + 1 < h ? (double)get(y + 1, x) : c;
    double lf = x > 0 ? (double)get(y, x - 1) : c;
    double rt = x + 1 < w ? (double)get(y, x + 1) : c;
    if (!finite_d(up)) up = c;
    if (!finite_d(dn)) dn = c;
    if (!finite_d(lf)) lf = c;
    if (!finite_d(rt)) rt = c;
    const double resp = dsub(dadd(dadd(dadd(up, dn), lf), rt), dmul(4.0, c));
    return fabs(resp) > dmul(thr, c);
}

// _native.pyx:205-220: reference depth of coarse pixel (cy,cx)
template <typename Get>
__device__ __forceinline__ double parent_ref_t(Get get, int64_t ch, int64_t cw, int64_t cy,
                                               int64_t cx, bool edge) {
    const double c = (double)get(cy, cx);
    double ref = finite_d(c) ? c : -INFINITY;
    if (edge) {
        for (int64_t ny = cy - 1; ny <= cy + 1; ++ny) {
            if (ny < 0 || ny >= ch) continue;
            for (int64_t nx = cx - 1; nx <= cx + 1; ++nx) {
                if (nx < 0 || nx >= cw || (ny == cy && nx == cx)) continue;
                const double v = (double)get(ny, nx);
                if (finite_d(v) && v > ref) ref = v;
            }
        }
    }
    return ref;
}

__device__ __forceinline__ bool keep_test(float f, double ref, double fs) {
    const double fd = (double)f;
    return finite_d(fd) && finite_d(ref) && dsub(fd, ref) <= dmul(fs, ref);
}

// _native.pyx:240-297 at one fine pixel (called only for holes)
template <typename Get>
__device__ __forceinline__ float bilinear_at_t(Get get, int64_t ch, int64_t cw, int64_t y,
                                               int64_t x) {
    const double gy = dsub(dmul(0.5, (double)y), 0.25);
    const int64_t y0r = (int64_t)floor(gy);
    const double wy1 = dsub(gy, (double)y0r), wy0 = dsub(1.0, wy1);
    const int64_t y0 = min(max(y0r, (int64_t)0), ch - 1), y1 = min(max(y0r + 1, (int64_t)0), ch - 1);
    const double gx = dsub(dmul(0.5, (double)x), 0.25);
    const int64_t x0r = (int64_t)floor(gx);
    const double wx1 = dsub(gx, (double)x0r), wx0 = dsub(1.0, wx1);
    const int64_t x0 = min(max(x0r, (int64_t)0), cw - 1), x1 = min(max(x0r + 1, (int64_t)0), cw - 1);
    double num = 0.0, den = 0.0;
    const int64_t yy[2] = {y0, y1};
    const int64_t xx[2] = {x0, x1};
    const double wy[2] = {wy0, wy1};
    const double wx[2] = {wx0, wx1};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const double v = (double)get(yy[a], xx[b]);
            if (finite_d(v)) {
                const double wgt = dmul(wy[a], wx[b]);
                num = dadd(num, dmul(wgt, v));
                den = dadd(den, wgt);
            }
        }
    }
    return den > 0.0 ? __double2float_rn(ddiv(num, den)) : INFINITY;
}

struct GlobalImg {
    const float *img;
    int64_t w;
    __device__ float operator()(int64_t y, int64_t x) const { return img[y * w + x]; }
};

__device__ __forceinline__ bool lap_edge(const float *__restrict__ img, int64_t h, int64_t w,
                                         int64_t y, int64_t x, double thr) {
    return lap_edge_t(GlobalImg{img, w}, h, w, y, x, thr);
}

__device__ __forceinline__ double parent_ref(const float *__restrict__ coarse, int64_t ch,
                                             int64_t cw, int64_t cy, int64_t cx, bool edge) {
    return parent_ref_t(GlobalImg{coarse, cw}, ch, cw, cy, cx, edge);
}

__device__ __forceinline__ float bilinear_at(const float *__restrict__ coarse, int64_t ch,
                                             int64_t cw, int64_t y, int64_t x) {
    return bilinear_at_t(GlobalImg{coarse, cw}, ch, cw, y, x);
}

// ----------------------------------------------------------------- twins ---

__global__ void k_min_pool(const float *__restrict__ img, int64_t h, int64_t w,
                           float *__restrict__ out) {
    const int64_t oh = (h + 1) / 2, ow = (w + 1) / 2;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < oh * ow;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = p / ow, x = p - y * ow;
        float m = INFINITY;
        for (int dy = 0; dy < 2; ++dy) {
            if (2 * y + dy >= h) break;
            for (int dx = 0; dx < 2; ++dx) {
                if (2 * x + dx >= w) break;
                const float v = img[(2 * y + dy) * w + 2 * x + dx];
                if (v < m) m = v;
            }
        }
        out[p] = m;
    }
}

__global__ void k_laplacian(const float *__restrict__ img, int64_t h, int64_t w, double thr,
                            uint8_t *__restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < h * w;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = p / w, x = p - y * w;
        out[p] = lap_edge(img, h, w, y, x, thr) ? 1 : 0;
    }
}

__global__ void k_keep(const float *__restrict__ coarse, int64_t ch, int64_t cw,
                       const uint8_t *__restrict__ edges, const float *__restrict__ fine,
                       int64_t fh, int64_t fw, double fs, float *__restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < fh * fw;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = p / fw, x = p - y * fw;
        const int64_t cy = y >> 1, cx = x >> 1;
        float o = INFINITY;
        if (cy < ch && cx < cw) {
            const double ref = parent_ref(coarse, ch, cw, cy, cx, edges[cy * cw + cx] != 0);
            if (keep_test(fine[p], ref, fs)) o = fine[p];
        }
        out[p] = o;
    }
}

__global__ void k_fill(const float *__restrict__ coarse, int64_t ch, int64_t cw,
                       const float *__restrict__ fine, int64_t fh, int64_t fw,
                       float *__restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < fh * fw;
         p += (int64_t)gridDim.x * blockDim.x) {
        const float f = fine[p];
        if (finite_f(f)) {
            out[p] = f;
        } else {
            const int64_t y = p / fw, x = p - y * fw;
            out[p] = bilinear_at(coarse, ch, cw, y, x);
        }
    }
}

// ---------------------------------------------------------- fused frame ---

struct Levels {
    float *img[8];  // pooled^1 .. pooled^L (index k-1)
    int64_t h[9], w[9];  // h[k] = size after k pools, k = 0..L
    int L;
};

// Writes one filtered pixel's U-Net input channels [r g b d' a 0 ...].
__device__ __forceinline__ void store_unet_px(__nv_bfloat16 *__restrict__ dst, int unet_c, float r,
                                              float g, float b, float dd, float a, double znear) {
    // weights.ts:90-95: d' = zNear/max(d, zNear) (f64 -> f32), 0 if empty
    const float dn = dd > 0.0f ? __double2float_rn(ddiv(znear, fmax((double)dd, znear))) : 0.0f;
    __nv_bfloat162 v01 = __floats2bfloat162_rn(r, g);
    __nv_bfloat162 v23 = __floats2bfloat162_rn(b, dn);
    __nv_bfloat162 v45 = __floats2bfloat162_rn(a, 0.0f);
    if ((unet_c & 7) == 0) {  // 16 B vector stores: [r g b d' | a 0 0 0 | 0 ...]
        uint4 *o4 = reinterpret_cast<uint4 *>(dst);
        o4[0] = make_uint4(*reinterpret_cast<uint32_t *>(&v01), *reinterpret_cast<uint32_t *>(&v23),
                           *reinterpret_cast<uint32_t *>(&v45), 0u);
        for (int c = 1; c < unet_c / 8; ++c) o4[c] = make_uint4(0u, 0u, 0u, 0u);
    } else {
        __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(dst);
        const __nv_bfloat162 z = __floats2bfloat162_rn(0.0f, 0.0f);
        o2[0] = v01;
        o2[1] = v23;
        o2[2] = v45;
        for (int c = 3; c < unet_c / 2; ++c) o2[c] = z;
    }
}

// 32x32 pixel block per CTA, 256 threads, 2x2 pixels per thread.
__global__ void __launch_bounds__(256) k_assemble_pyramid(
    unsigned long long *__restrict__ minz, float4 *__restrict__ acc, int64_t H,
    int64_t W, Levels lv, int pool_levels, float *__restrict__ rgb, float *__restrict__ depth,
    uint8_t *__restrict__ alpha, int *__restrict__ flags, __nv_bfloat16 *__restrict__ unet_in,
    int unet_c, double znear) {
    pdl_wait();  // launched with PDL after pass 2; its trigger is completion
    __shared__ float s1[16][17];
    __shared__ float s2[8][9];
    __shared__ float s3[4][5];
    __shared__ float s4[2][3];
    const int gy = threadIdx.x >> 4, gx = threadIdx.x & 15;
    const int64_t by = blockIdx.y, bx = blockIdx.x;
    float m = INFINITY;
    bool overflow = false;
    const int64_t x = bx * 32 + 2 * gx;
    // Issue every load of the thread's 2x2 pixels before any use (4 independent
    // 8 B minz + 16 B accum pairs in flight), then compute, then vector stores.
    unsigned long long key[2][2];
    float4 a[2][2];
    bool ok[2][2];
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int64_t y = by * 32 + 2 * gy + dy;
        const int64_t p = y * W + x;
        ok[dy][0] = y < H && x < W;
        ok[dy][1] = y < H && x + 1 < W;
        if (ok[dy][1] && (W & 1) == 0) {
            const ulonglong2 k2 = __ldcs(reinterpret_cast<const ulonglong2 *>(minz + p));
            key[dy][0] = k2.x; key[dy][1] = k2.y;
            a[dy][0] = acc[p];
            a[dy][1] = acc[p + 1];
        } else {
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                key[dy][dx] = ok[dy][dx] ? minz[p + dx] : kInfBits;
                a[dy][dx] = ok[dy][dx] ? acc[p + dx] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int64_t y = by * 32 + 2 * gy + dy;
        const int64_t p = y * W + x;
        float c[2][3], d[2];
        uint8_t al[2];
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            // the f32 sums are exact integers while every field stays < 2^24
            // (any partial sum reaching 2^24 leaves the final field >= 2^24)
            const float4 f = a[dy][dx];
            d[dx] = 0.0f;
            c[dx][0] = c[dx][1] = c[dx][2] = 0.0f;
            al[dx] = 0;
            if (f.w > 0.0f) {
                overflow |= fmaxf(fmaxf(f.x, f.y), fmaxf(f.z, f.w)) >= kAccumExactLimit;
                // render.py:146-161 computes f32(f64(sum) / (f64(count) * 255)).
                // With integer sum < 2^24, d = count * 255 < 2^24 (exact in f32)
                // and sum / d <= 1, the f32 IEEE division gives the same bits:
                // RN64 then RN32 can differ from RN32 only if RN64(v) hits an
                // f32 midpoint m != v, but |v - m| >= 2^(E-24) / d > ulp64(m) / 2
                // for v < 2^25 (tests/test_oracle_golden.py checks the identity
                // exhaustively for small counts and on 1e8 random pairs).  Three
                // f32 divisions instead of three f64 ones.
                const float denom = __fmul_rn(f.w, 255.0f);
                c[dx][0] = __fdiv_rn(f.x, denom);
                c[dx][1] = __fdiv_rn(f.y, denom);
                c[dx][2] = __fdiv_rn(f.z, denom);
                d[dx] = __double2float_rn(__longlong_as_double((long long)key[dy][dx]));
                al[dx] = 1;
            }
            if (ok[dy][dx]) {
                const float sv = sentinel(d[dx]);
                m = sv < m ? sv : m;
            }
        }
        if (unet_in) {
            // U-Net-only frames: the input of every pixel as if kept (the
            // final filter step clears the rejected ones) -- no f32 rgb round trip
#pragma unroll
            for (int dx = 0; dx < 2; ++dx)
                if (ok[dy][dx])
                    store_unet_px(unet_in + (p + dx) * unet_c, unet_c, c[dx][0], c[dx][1], c[dx][2],
                                  d[dx], (float)al[dx], znear);
        }
        if (ok[dy][1] && (W & 1) == 0) {
            if (rgb) {
                float2 *r2 = reinterpret_cast<float2 *>(rgb + 3 * p);
                r2[0] = make_float2(c[0][0], c[0][1]);
                r2[1] = make_float2(c[0][2], c[1][0]);
                r2[2] = make_float2(c[1][1], c[1][2]);
            }
            *reinterpret_cast<float2 *>(depth + p) = make_float2(d[0], d[1]);
            if (alpha) *reinterpret_cast<uchar2 *>(alpha + p) = make_uchar2(al[0], al[1]);
            // consume-and-reset for the next frame
            *reinterpret_cast<ulonglong2 *>(minz + p) = make_ulonglong2(kInfBits, kInfBits);
            acc[p] = make_float4(0.f, 0.f, 0.f, 0.f);
            acc[p + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                if (!ok[dy][dx]) continue;
                const int64_t q = p + dx;
                if (rgb) {
                    rgb[3 * q] = c[dx][0];
                    rgb[3 * q + 1] = c[dx][1];
                    rgb[3 * q + 2] = c[dx][2];
                }
                depth[q] = d[dx];
                if (alpha) alpha[q] = al[dx];
                minz[q] = kInfBits;
                acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    if (overflow) atomicOr(flags, 1);
    if (pool_levels < 1) return;
    // level 1
    {
        const int64_t y = by * 16 + gy, x = bx * 16 + gx;
        if (y < lv.h[1] && x < lv.w[1]) lv.img[0][y * lv.w[1] + x] = m;
        s1[gy][gx] = m;  // out-of-image entries are +inf == skipped children
    }
    if (pool_levels < 2) return;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int ty = threadIdx.x >> 3, tx = threadIdx.x & 7;
        float v = fminf(fminf(s1[2 * ty][2 * tx], s1[2 * ty][2 * tx + 1]),
                        fminf(s1[2 * ty + 1][2 * tx], s1[2 * ty + 1][2 * tx + 1]));
        s2[ty][tx] = v;
        const int64_t y = by * 8 + ty, x = bx * 8 + tx;
        if (y < lv.h[2] && x < lv.w[2]) lv.img[1][y * lv.w[2] + x] = v;
    }
    if (pool_levels < 3) return;
    __syncthreads();
    if (threadIdx.x < 16) {
        const int ty = threadIdx.x >> 2, tx = threadIdx.x & 3;
        float v = fminf(fminf(s2[2 * ty][2 * tx], s2[2 * ty][2 * tx + 1]),
                        fminf(s2[2 * ty + 1][2 * tx], s2[2 * ty + 1][2 * tx + 1]));
        s3[ty][tx] = v;
        const int64_t y = by * 4 + ty, x = bx * 4 + tx;
        if (y < lv.h[3] && x < lv.w[3]) lv.img[2][y * lv.w[3] + x] = v;
    }
    if (pool_levels < 4) return;
    __syncthreads();
    if (threadIdx.x < 4) {
        const int ty = threadIdx.x >> 1, tx = threadIdx.x & 1;
        float v = fminf(fminf(s3[2 * ty][2 * tx], s3[2 * ty][2 * tx + 1]),
                        fminf(s3[2 * ty + 1][2 * tx], s3[2 * ty + 1][2 * tx + 1]));
        s4[ty][tx] = v;
        const int64_t y = by * 2 + ty, x = bx * 2 + tx;
        if (y < lv.h[4] && x < lv.w[4]) lv.img[3][y * lv.w[4] + x] = v;
    }
    if (pool_levels < 5) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = fminf(fminf(s4[0][0], s4[0][1]), fminf(s4[1][0], s4[1][1]));
        if (by < lv.h[5] && bx < lv.w[5]) lv.img[4][by * lv.w[5] + bx] = v;
    }
}

// Arguments of the final (full-resolution) filter step.
struct FinalArgs {
    const float *fine;  // frame depth (0 = empty)
    int64_t fh, fw;
    const float *rgb;
    const uint8_t *alpha;
    float *frgb, *fdepth;
    uint8_t *falpha, *keep;
    __nv_bfloat16 *unet_in;
    int unet_c;
    double znear;
};

// The final step for the 2x2 children of coarse pixel (cy, cx) given its
// reference depth: keep mask, filtered frame and / or U-Net input.  Where the
// two children of a fine row are both inside an even-width image they move
// with 8 B (rgb, depth), 2 B (alpha) and 16 B (U-Net) accesses.
__device__ __forceinline__ void final_children(const FinalArgs &fa, int64_t cy, int64_t cx,
                                               double ref, double fs) {
    const int64_t fh = fa.fh, fw = fa.fw;
    const float *__restrict__ fine = fa.fine;
    const float *__restrict__ rgb = fa.rgb;
    const int64_t x = 2 * cx;
    const bool pair = x + 1 < fw && (fw & 1) == 0;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int64_t y = 2 * cy + dy;
        if (y >= fh) break;
        const int64_t p = y * fw + x;
        if (!pair) {  // odd width or the last column: scalar children
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                if (x + dx >= fw) break;
                const int64_t q = p + dx;
                const float dq = fine[q];  // frame depth (0 = empty)
                const bool kq = keep_test(sentinel(dq), ref, fs);
                if (fa.keep) fa.keep[q] = (uint8_t)kq;
                if (!rgb) {  // mask-only, or U-Net-only: clear a rejected non-empty pixel
                    if (fa.unet_in && !kq && dq > 0.0f)
                        store_unet_px(fa.unet_in + q * fa.unet_c, fa.unet_c, 0.f, 0.f, 0.f, 0.f,
                                      0.f, fa.znear);
                    continue;
                }
                const float m = kq ? 1.0f : 0.0f;  // filtering.py:141-147 f32 0/1 mask
                const float r = rgb[3 * q] * m, g = rgb[3 * q + 1] * m, b = rgb[3 * q + 2] * m,
                            dd = dq * m;
                const uint8_t a = (uint8_t)(fa.alpha[q] * (uint8_t)kq);
                if (fa.frgb) {
                    fa.frgb[3 * q] = r;
                    fa.frgb[3 * q + 1] = g;
                    fa.frgb[3 * q + 2] = b;
                }
                if (fa.fdepth) fa.fdepth[q] = dd;
                if (fa.falpha) fa.falpha[q] = a;
                if (fa.unet_in)
                    store_unet_px(fa.unet_in + q * fa.unet_c, fa.unet_c, r, g, b, dd, a, fa.znear);
            }
            continue;
        }
        const float2 d2 = *reinterpret_cast<const float2 *>(fine + p);
        const float d[2] = {d2.x, d2.y};
        bool k[2];
        float mk[2];
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            k[dx] = keep_test(sentinel(d[dx]), ref, fs);
            mk[dx] = k[dx] ? 1.0f : 0.0f;
        }
        if (fa.keep) *reinterpret_cast<uchar2 *>(fa.keep + p) = make_uchar2(k[0], k[1]);
        if (!rgb) {
            if (fa.unet_in) {
#pragma unroll
                for (int dx = 0; dx < 2; ++dx)
                    if (!k[dx] && d[dx] > 0.0f)
                        store_unet_px(fa.unet_in + (p + dx) * fa.unet_c, fa.unet_c, 0.f, 0.f, 0.f,
                                      0.f, 0.f, fa.znear);
            }
            continue;
        }
        const float2 *r2 = reinterpret_cast<const float2 *>(rgb + 3 * p);
        const float2 a0 = r2[0], a1 = r2[1], a2 = r2[2];
        const float c[2][3] = {{a0.x, a0.y, a1.x}, {a1.y, a2.x, a2.y}};
        const uchar2 a2v = *reinterpret_cast<const uchar2 *>(fa.alpha + p);
        const uint8_t al[2] = {a2v.x, a2v.y};
        float o[2][4];
        uint8_t oa[2];
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            o[dx][0] = c[dx][0] * mk[dx];
            o[dx][1] = c[dx][1] * mk[dx];
            o[dx][2] = c[dx][2] * mk[dx];
            o[dx][3] = d[dx] * mk[dx];
            oa[dx] = (uint8_t)(al[dx] * (uint8_t)k[dx]);
        }
        if (fa.frgb) {
            float2 *w2 = reinterpret_cast<float2 *>(fa.frgb + 3 * p);
            w2[0] = make_float2(o[0][0], o[0][1]);
            w2[1] = make_float2(o[0][2], o[1][0]);
            w2[2] = make_float2(o[1][1], o[1][2]);
        }
        if (fa.fdepth) *reinterpret_cast<float2 *>(fa.fdepth + p) = make_float2(o[0][3], o[1][3]);
        if (fa.falpha) *reinterpret_cast<uchar2 *>(fa.falpha + p) = make_uchar2(oa[0], oa[1]);
        if (fa.unet_in) {
#pragma unroll
            for (int dx = 0; dx < 2; ++dx)
                store_unet_px(fa.unet_in + (p + dx) * fa.unet_c, fa.unet_c, o[dx][0], o[dx][1],
                              o[dx][2], o[dx][3], oa[dx], fa.znear);
        }
    }
}

// One thread per COARSE pixel on a 2-D grid (32 x 8 threads per CTA, no
// index division); FINAL reads the full-resolution frame (final_children).
template <bool FINAL>
__global__ void __launch_bounds__(256) k_filter_step(
    const float *__restrict__ coarse, int64_t ch, int64_t cw, const float *__restrict__ fine,
    int64_t fh, int64_t fw, double fs, double et, float *__restrict__ out, FinalArgs fa) {
    pdl_wait();
    const int64_t cx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t cy = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
    if (cx >= cw || cy >= ch) return;
    const bool edge = lap_edge(coarse, ch, cw, cy, cx, et);
    const double ref = parent_ref(coarse, ch, cw, cy, cx, edge);
    if (FINAL) {
        final_children(fa, cy, cx, ref, fs);
    } else {
        const int64_t x = 2 * cx;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
            const int64_t y = 2 * cy + dy;
            if (y >= fh) break;
            const int64_t p = y * fw + x;
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                if (x + dx >= fw) break;
                const float f = fine[p + dx];
                out[p + dx] = keep_test(f, ref, fs) ? f : bilinear_at(coarse, ch, cw, y, x + dx);
            }
        }
    }
    pdl_trigger();
}

// Bridge input (FE:bridge.ts:31-53): an RGDA tensor's five f32 planes ->
// the U-Net's bf16 NHWC input, one thread per pixel.
__global__ void __launch_bounds__(256) k_pack_rgbda(const float *__restrict__ planes, int64_t n_px,
                                                    int64_t width, __nv_bfloat16 *__restrict__ out,
                                                    int unet_c, double znear) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_px;
         i += (int64_t)gridDim.x * blockDim.x)
        store_unet_px(out + i * unet_c, unet_c, planes[i], planes[n_px + i], planes[2 * n_px + i],
                      planes[3 * n_px + i], planes[4 * n_px + i], znear);
}

inline dim3 step_grid2(int64_t ch, int64_t cw) {
    return dim3((unsigned)((cw + 31) / 32), (unsigned)((ch + 7) / 8));
}

inline void level_sizes(int64_t H, int64_t W, int L, int64_t *h, int64_t *w) {
    h[0] = H;
    w[0] = W;
    for (int k = 1; k <= L; ++k) {
        h[k] = (h[k - 1] + 1) / 2;
        w[k] = (w[k - 1] + 1) / 2;
    }
}

// ---- fused non-final steps ------------------------------------------------
// All L-1 non-final steps of the filter in ONE launch (filtering.py:124-131):
// each CTA produces a 64x32 tile of the last non-final step's output and
// recomputes, in shared memory, exactly the parts of the coarser steps' outputs
// its stencils read (every output pixel depends on a 3x3 coarse window, so a
// level-k region needs its parents +-1 at level k+1).  Neighbouring CTAs
// recompute overlapping halos with the same arithmetic, so the result is the
// per-step kernels' bit for bit; the L-1 launches (each latency-bound on a
// small image) become one.
// (FINAL: the last non-final level is produced on the tile +- 1, 34 x 18 values)
constexpr int kFuseTX = 32, kFuseTY = 16, kFuseMaxSteps = 4, kFuseBuf = 640;

struct Rect {
    int y0, y1, x0, x1;  // [y0, y1) x [x0, x1)
    __device__ int h() const { return y1 - y0; }
    __device__ int w() const { return x1 - x0; }
};

// the coarse pixels a fine region's stencils read: parents +-1, clipped
__device__ __forceinline__ Rect coarse_of(const Rect &f, int ch, int cw) {
    Rect c;
    c.y0 = max((f.y0 >> 1) - 1, 0);
    c.y1 = min(((f.y1 - 1) >> 1) + 2, ch);
    c.x0 = max((f.x0 >> 1) - 1, 0);
    c.x1 = min(((f.x1 - 1) >> 1) + 2, cw);
    return c;
}

struct SmemImg {
    const float *buf;
    Rect r;
    __device__ float operator()(int64_t y, int64_t x) const {
        return buf[((int)y - r.y0) * r.w() + ((int)x - r.x0)];
    }
};

// filter_strength per blockIdx.z: a sweep over strengths runs every strength's
// steps in one launch (the pyramid they read is strength-independent); output
// z lands at out + z * out_stride.
constexpr int kMaxSweep = 16;
struct FsSweep {
    double fs[kMaxSweep];
    int64_t out_stride;
};

// FINAL: the final (full-resolution) step fused in as well -- the last
// non-final step is produced on the tile +- 1 (the final step's 3x3 stencils)
// into shared memory, then every level-1 pixel of the tile runs the final
// step for its 2x2 children (final_children, the arithmetic of
// k_filter_step<true>), so the whole filter after the pyramid is one launch.
template <bool FINAL>
__global__ void __launch_bounds__(256) k_filter_coarse_fused(Levels lv, float *__restrict__ out,
                                                             FsSweep sw, double et, FinalArgs fa) {
    pdl_wait();
    const double fs = sw.fs[blockIdx.z];
    out += blockIdx.z * sw.out_stride;
    __shared__ float ubuf[2][kFuseBuf];     // coarse input of the current step / its output
    __shared__ double refbuf[kFuseBuf];     // reference depth per parent pixel
    const int L = lv.L, nsteps = L - 1;
    // regions: R[i] = output region of step i+1 (level L-1-i), R[nsteps-1] = this tile
    // (FINAL: the tile +- 1)
    Rect R[kFuseMaxSteps];
    Rect t;
    t.y0 = blockIdx.y * kFuseTY;
    t.y1 = min(t.y0 + kFuseTY, (int)lv.h[1]);
    t.x0 = blockIdx.x * kFuseTX;
    t.x1 = min(t.x0 + kFuseTX, (int)lv.w[1]);
    {
        Rect r = t;
        if (FINAL) {
            r.y0 = max(t.y0 - 1, 0);
            r.y1 = min(t.y1 + 1, (int)lv.h[1]);
            r.x0 = max(t.x0 - 1, 0);
            r.x1 = min(t.x1 + 1, (int)lv.w[1]);
        }
        R[nsteps - 1] = r;
        for (int i = nsteps - 2; i >= 0; --i)  // R[i] lies on level L-1-i
            R[i] = coarse_of(R[i + 1], (int)lv.h[L - 1 - i], (int)lv.w[L - 1 - i]);
    }
    // coarse input of step 1: pooled^L on coarse_of(R[0])
    Rect C = coarse_of(R[0], (int)lv.h[L], (int)lv.w[L]);
    int cur = 0;
    for (int i = threadIdx.x; i < C.h() * C.w(); i += blockDim.x) {
        const int y = C.y0 + i / C.w(), x = C.x0 + i % C.w();
        ubuf[cur][i] = lv.img[L - 1][(int64_t)y * lv.w[L] + x];
    }
    __syncthreads();
    for (int st = 0; st < nsteps; ++st) {
        const int clev = L - st, flev = L - st - 1;  // coarse / fine levels of this step
        const int64_t ch = lv.h[clev], cw = lv.w[clev], fw = lv.w[flev];
        const float *fine = lv.img[flev - 1];        // pooled^flev
        const Rect F = R[st];
        const SmemImg getC{ubuf[cur], C};
        // parents of F (inside C by construction)
        Rect P;
        P.y0 = F.y0 >> 1;
        P.y1 = ((F.y1 - 1) >> 1) + 1;
        P.x0 = F.x0 >> 1;
        P.x1 = ((F.x1 - 1) >> 1) + 1;
        for (int i = threadIdx.x; i < P.h() * P.w(); i += blockDim.x) {
            const int cy = P.y0 + i / P.w(), cx = P.x0 + i % P.w();
            const bool edge = lap_edge_t(getC, ch, cw, cy, cx, et);
            refbuf[i] = parent_ref_t(getC, ch, cw, cy, cx, edge);
        }
        __syncthreads();
        const bool last = st == nsteps - 1;
        for (int i = threadIdx.x; i < F.h() * F.w(); i += blockDim.x) {
            const int y = F.y0 + i / F.w(), x = F.x0 + i % F.w();
            const double ref = refbuf[((y >> 1) - P.y0) * P.w() + ((x >> 1) - P.x0)];
            const float f = fine[(int64_t)y * fw + x];
            const float o = keep_test(f, ref, fs) ? f : bilinear_at_t(getC, ch, cw, y, x);
            if (!last || FINAL) ubuf[cur ^ 1][i] = o;
            if (last && (!FINAL || (y >= t.y0 && y < t.y1 && x >= t.x0 && x < t.x1)))
                out[(int64_t)y * fw + x] = o;
        }
        __syncthreads();
        cur ^= 1;
        C = F;
    }
    if (FINAL) {
        // the final step's coarse image is level 1 on C (= the tile +- 1)
        const int64_t ch = lv.h[1], cw = lv.w[1];
        const SmemImg getC{ubuf[cur], C};
        for (int i = threadIdx.x; i < t.h() * t.w(); i += blockDim.x) {
            const int cy = t.y0 + i / t.w(), cx = t.x0 + i % t.w();
            const bool edge = lap_edge_t(getC, ch, cw, cy, cx, et);
            final_children(fa, cy, cx, parent_ref_t(getC, ch, cw, cy, cx, edge), fs);
        }
    }
    pdl_trigger();
}

// Does a fused coarse launch cover this pyramid?  (every intermediate region
// must fit the shared buffers: true for kFuseTY x kFuseTX tiles and L <= 5)
inline bool fused_ok(const Levels &lv) { return lv.L >= 2 && lv.L - 1 <= kFuseMaxSteps; }

// LS_FILTER_FUSED (A/B measurements): 0 = one launch per step, 1 (default) =
// the non-final steps in one launch + the final step, 2 = all steps in one
// launch (measured slower at 1080p: 807 vs 813 frames/s -- the fused final
// step runs 2048 pixels per 256-thread CTA after the coarse steps, the
// separate one 4 pixels per thread over the whole frame).
inline int fused_mode() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_FILTER_FUSED");
        r = (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r;
}

// Pyramid + steps over an existing sentinel-able depth image.  `lvl` holds
// pooled^1..pooled^L, `up` the filled images of steps 1..L-1.
int run_filter_steps(const Levels &lv, float *up_base, const float *full_fine, int64_t H,
                     int64_t W, double fs, double et, float *keep_as_out, const float *rgb,
                     const uint8_t *alpha, float *frgb, float *fdepth, uint8_t *falpha,
                     uint8_t *keep, __nv_bfloat16 *unet_in, int unet_c, double znear,
                     cudaStream_t st) {
    const int L = lv.L;
    const float *coarse = lv.img[L - 1];  // pyr.levels[0]
    float *up = up_base;
    int first = 1;
    const FinalArgs fa{full_fine, H, W, rgb, alpha, frgb, fdepth, falpha, keep, unet_in, unet_c, znear};
    if (fused_ok(lv) && fused_mode() >= 1) {
        // steps 1..L-1 in one launch; its output sits where step L-1 would write
        // (mode 2: the final step in the same launch)
        for (int i = 1; i < L - 1; ++i) up += lv.h[L - i] * lv.w[L - i];
        const dim3 g((unsigned)((lv.w[1] + kFuseTX - 1) / kFuseTX),
                     (unsigned)((lv.h[1] + kFuseTY - 1) / kFuseTY));
        FsSweep sw{};
        sw.fs[0] = fs;
        const bool all = fused_mode() == 2;
        cudaError_t e = all ? launch_pdl(k_filter_coarse_fused<true>, g, dim3(256), 0, st, lv, up,
                                         sw, et, fa)
                            : launch_pdl(k_filter_coarse_fused<false>, g, dim3(256), 0, st, lv, up,
                                         sw, et, FinalArgs{});
        if (e != cudaSuccess) return (int)e;
        if (all) return 0;
        coarse = up;
        up += lv.h[1] * lv.w[1];
        first = L;
    }
    for (int i = first; i <= L; ++i) {
        const int64_t ch = lv.h[L - i + 1], cw = lv.w[L - i + 1];
        const int64_t fh = lv.h[L - i], fw = lv.w[L - i];
        if (i < L) {
            const float *fine = lv.img[L - i - 1];
            cudaError_t e = launch_pdl(k_filter_step<false>, step_grid2(ch, cw), dim3(32, 8), 0, st,
                                       coarse, ch, cw, fine, fh, fw, fs, et, up, FinalArgs{});
            if (e != cudaSuccess) return (int)e;
            coarse = up;
            up += fh * fw;
        } else {
            cudaError_t e = launch_pdl(k_filter_step<true>, step_grid2(ch, cw), dim3(32, 8), 0, st,
                                       coarse, ch, cw, full_fine, fh, fw, fs, et, keep_as_out, fa);
            if (e != cudaSuccess) return (int)e;
        }
    }
    return 0;
}

__global__ void k_to_sentinel_pool(const float *__restrict__ depth, int64_t h, int64_t w,
                                   float *__restrict__ out) {
    const int64_t oh = (h + 1) / 2, ow = (w + 1) / 2;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < oh * ow;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = p / ow, x = p - y * ow;
        float m = INFINITY;
        for (int dy = 0; dy < 2; ++dy) {
            if (2 * y + dy >= h) break;
            for (int dx = 0; dx < 2; ++dx) {
                if (2 * x + dx >= w) break;
                const float v = sentinel(depth[(2 * y + dy) * w + 2 * x + dx]);
                if (v < m) m = v;
            }
        }
        out[p] = m;
    }
}

// Final step of a filter_strength sweep (C4): one thread per
// coarse pixel reads its <= 4 children's frame values ONCE and, for each of
// the nk strengths, runs the edge / reference / keep test against that
// strength's coarse image (coarse0 + k * cstride) and writes the k-th keep
// mask and filtered frame (outputs at + k * fh * fw).  Same arithmetic as
// k_filter_step<true>, so every strength's outputs equal a single-strength
// depth filter bit for bit.
__global__ void __launch_bounds__(256) k_filter_final_sweep(
    const float *__restrict__ coarse0, int64_t cstride, int64_t ch, int64_t cw,
    const float *__restrict__ depth, const float *__restrict__ rgb,
    const uint8_t *__restrict__ alpha, int64_t fh, int64_t fw, FsSweep sw, int nk, double et,
    float *__restrict__ frgb, float *__restrict__ fdepth, uint8_t *__restrict__ falpha,
    uint8_t *__restrict__ keep_out) {
    pdl_wait();
    const int64_t cx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t cy = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
    if (cx >= cw || cy >= ch) return;
    const int64_t x = 2 * cx;
    // both children of a row move as one 8 B (depth, rgb) / 2 B (alpha, keep)
    // access when the width is even (the common case); else per child
    const bool pair = x + 1 < fw && (fw & 1) == 0;
    float d[2][2], c[2][2][3];
    uint8_t a[2][2];
    int rows = 0;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int64_t y = 2 * cy + dy;
        if (y >= fh) break;
        ++rows;
        const int64_t p = y * fw + x;
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            const bool in = x + dx < fw;
            d[dy][dx] = in ? depth[p + dx] : 0.0f;
            if (rgb) {
#pragma unroll
                for (int q = 0; q < 3; ++q) c[dy][dx][q] = in ? rgb[3 * (p + dx) + q] : 0.0f;
                a[dy][dx] = in ? alpha[p + dx] : (uint8_t)0;
            }
        }
    }
    const int64_t hw = fh * fw;
    for (int k = 0; k < nk; ++k) {
        const float *coarse = coarse0 + k * cstride;
        const bool edge = lap_edge(coarse, ch, cw, cy, cx, et);
        const double ref = parent_ref(coarse, ch, cw, cy, cx, edge);
        const double fs = sw.fs[k];
        for (int dy = 0; dy < rows; ++dy) {
            const int64_t o = k * hw + (2 * cy + dy) * fw + x;
            bool kq[2];
            float m[2];
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                kq[dx] = keep_test(sentinel(d[dy][dx]), ref, fs);
                m[dx] = kq[dx] ? 1.0f : 0.0f;  // filtering.py:141-147 f32 0/1 mask
            }
            if (pair) {
                if (keep_out) *reinterpret_cast<uchar2 *>(keep_out + o) = make_uchar2(kq[0], kq[1]);
                if (!rgb) continue;
                if (frgb) {
                    float2 *w2 = reinterpret_cast<float2 *>(frgb + 3 * o);
                    w2[0] = make_float2(c[dy][0][0] * m[0], c[dy][0][1] * m[0]);
                    w2[1] = make_float2(c[dy][0][2] * m[0], c[dy][1][0] * m[1]);
                    w2[2] = make_float2(c[dy][1][1] * m[1], c[dy][1][2] * m[1]);
                }
                if (fdepth)
                    *reinterpret_cast<float2 *>(fdepth + o) =
                        make_float2(d[dy][0] * m[0], d[dy][1] * m[1]);
                if (falpha)
                    *reinterpret_cast<uchar2 *>(falpha + o) =
                        make_uchar2((uint8_t)(a[dy][0] * (uint8_t)kq[0]),
                                    (uint8_t)(a[dy][1] * (uint8_t)kq[1]));
                continue;
            }
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                if (x + dx >= fw) break;
                if (keep_out) keep_out[o + dx] = (uint8_t)kq[dx];
                if (!rgb) continue;
                if (frgb) {
                    frgb[3 * (o + dx)] = c[dy][dx][0] * m[dx];
                    frgb[3 * (o + dx) + 1] = c[dy][dx][1] * m[dx];
                    frgb[3 * (o + dx) + 2] = c[dy][dx][2] * m[dx];
                }
                if (fdepth) fdepth[o + dx] = d[dy][dx] * m[dx];
                if (falpha) falpha[o + dx] = (uint8_t)(a[dy][dx] * (uint8_t)kq[dx]);
            }
        }
    }
    pdl_trigger();
}

bool setup_levels(int64_t H, int64_t W, int L, float *pyr, Levels &lv, float *&up_base) {
    if (L < 1 || L > 8) return false;
    if (H < (int64_t(1) << L) || W < (int64_t(1) << L)) return false;  // filtering.py:75-78
    lv.L = L;
    level_sizes(H, W, L, lv.h, lv.w);
    float *p = pyr;
    for (int k = 1; k <= L; ++k) {
        lv.img[k - 1] = p;
        p += lv.h[k] * lv.w[k];
    }
    up_base = p;
    return true;
}

}  // namespace ls

using namespace ls;

extern "C" {

int ls_min_pool_2x2(const float *d_img, int64_t h, int64_t w, float *d_out, void *stream) {
    if (h <= 0 || w <= 0) return LS_EINVAL;
    const int64_t n = ((h + 1) / 2) * ((w + 1) / 2);
    k_min_pool<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(d_img, h, w, d_out);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_laplacian_edges(const float *d_img, int64_t h, int64_t w, double threshold,
                       uint8_t *d_out, void *stream) {
    if (h <= 0 || w <= 0) return LS_EINVAL;
    k_laplacian<<<grid_for(h * w, 256), 256, 0, (cudaStream_t)stream>>>(d_img, h, w, threshold,
                                                                        d_out);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_filter_keep(const float *d_coarse, int64_t ch, int64_t cw, const uint8_t *d_edges,
                   const float *d_fine, int64_t fh, int64_t fw, double filter_strength,
                   float *d_out, void *stream) {
    if (ch <= 0 || cw <= 0 || fh <= 0 || fw <= 0) return LS_EINVAL;
    k_keep<<<grid_for(fh * fw, 256), 256, 0, (cudaStream_t)stream>>>(
        d_coarse, ch, cw, d_edges, d_fine, fh, fw, filter_strength, d_out);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_bilinear_fill(const float *d_coarse, int64_t ch, int64_t cw, const float *d_fine,
                     int64_t fh, int64_t fw, float *d_out, void *stream) {
    if (ch <= 0 || cw <= 0 || fh <= 0 || fw <= 0) return LS_EINVAL;
    k_fill<<<grid_for(fh * fw, 256), 256, 0, (cudaStream_t)stream>>>(d_coarse, ch, cw, d_fine,
                                                                     fh, fw, d_out);
    LS_LAUNCH_CHECK();
    return 0;
}

int64_t ls_pyramid_floats(int64_t height, int64_t width, int32_t levels_n) {
    if (levels_n < 1 || levels_n > 8 || height <= 0 || width <= 0) return -1;
    int64_t h[9], w[9];
    level_sizes(height, width, levels_n, h, w);
    int64_t total = 0;
    for (int k = 1; k <= levels_n; ++k) total += 2 * h[k] * w[k];
    return total;
}

int ls_frame_finish(uint64_t *d_minz_bits, float *d_accum4, int64_t width, int64_t height,
                    const ls_filter_params *filter, float *d_rgb, float *d_depth,
                    uint8_t *d_alpha, float *d_frgb, float *d_fdepth, uint8_t *d_falpha,
                    uint8_t *d_keep, uint16_t *d_unet_in, int64_t unet_h, int32_t unet_c,
                    double unet_znear, float *d_pyramid, int32_t *d_flags, void *stream) {
    // U-Net-only frames (a filter, a U-Net input, no raw rgb/alpha and no
    // filtered outputs): the assembly writes the U-Net input of every pixel and
    // the final filter step only clears the rejected ones
    const bool unet_only = filter && d_unet_in && !d_rgb && !d_alpha && !d_frgb && !d_fdepth &&
                           !d_falpha;
    if (width <= 0 || height <= 0 || !d_depth || !d_flags) return LS_EINVAL;
    if (!unet_only && (!d_rgb || !d_alpha)) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Levels lv{};
    float *up_base = nullptr;
    int L = 0;
    if (filter) {
        if (!d_pyramid || filter->filter_strength < 0 || filter->edge_threshold <= 0)
            return LS_EINVAL;
        if (!setup_levels(height, width, filter->levels_n, d_pyramid, lv, up_base))
            return LS_EINVAL;
        if (d_unet_in && (unet_h < height || unet_c < 6 || (unet_c & 1))) return LS_EINVAL;
        L = filter->levels_n;
    }
    dim3 grid((unsigned)((width + 31) / 32), (unsigned)((height + 31) / 32));
    const int in_block = L < 5 ? L : 5;
    cudaError_t e = launch_pdl(k_assemble_pyramid, grid, dim3(256), 0, st,
                               (unsigned long long *)d_minz_bits,
                               reinterpret_cast<float4 *>(d_accum4), height, width, lv, in_block,
                               d_rgb, d_depth, d_alpha, d_flags,
                               unet_only ? reinterpret_cast<__nv_bfloat16 *>(d_unet_in) : nullptr,
                               (int)unet_c, unet_znear);
    if (e != cudaSuccess) return (int)e;
    if (!filter) return 0;
    for (int k = 6; k <= L; ++k) {  // levels beyond the in-block five
        k_min_pool<<<grid_for(lv.h[k] * lv.w[k], 256), 256, 0, st>>>(lv.img[k - 2], lv.h[k - 1],
                                                                     lv.w[k - 1], lv.img[k - 1]);
        LS_LAUNCH_CHECK();
    }
    return run_filter_steps(lv, up_base, d_depth, height, width, filter->filter_strength,
                            filter->edge_threshold, nullptr, d_rgb, d_alpha, d_frgb, d_fdepth,
                            d_falpha, d_keep, reinterpret_cast<__nv_bfloat16 *>(d_unet_in),
                            unet_c, unet_znear, st);
}

int ls_unet_pack_rgbda(const float *d_planes, int64_t height, int64_t width, int32_t unet_c,
                       double unet_znear, uint16_t *d_unet_in, void *stream) {
    if (!d_planes || !d_unet_in || height <= 0 || width <= 0 || unet_c < 6 || (unet_c & 1) ||
        !(unet_znear > 0.0))
        return LS_EINVAL;
    if ((unet_c & 7) == 0 && (reinterpret_cast<uintptr_t>(d_unet_in) & 15)) return LS_EINVAL;
    const int64_t n = height * width;
    k_pack_rgbda<<<grid_for(n, 256, 8), 256, 0, (cudaStream_t)stream>>>(
        d_planes, n, width, reinterpret_cast<__nv_bfloat16 *>(d_unet_in), unet_c, unet_znear);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_filter_depth_image(const float *d_depth, int64_t height, int64_t width,
                          const ls_filter_params *filter, uint8_t *d_keep, float *d_pyramid,
                          void *stream) {
    if (!filter || !d_keep || !d_pyramid || height <= 0 || width <= 0) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Levels lv{};
    float *up_base = nullptr;
    if (!setup_levels(height, width, filter->levels_n, d_pyramid, lv, up_base)) return LS_EINVAL;
    const int L = lv.L;
    k_to_sentinel_pool<<<grid_for(lv.h[1] * lv.w[1], 256), 256, 0, st>>>(d_depth, height, width,
                                                                         lv.img[0]);
    LS_LAUNCH_CHECK();
    for (int k = 2; k <= L; ++k) {
        k_min_pool<<<grid_for(lv.h[k] * lv.w[k], 256), 256, 0, st>>>(lv.img[k - 2], lv.h[k - 1],
                                                                     lv.w[k - 1], lv.img[k - 1]);
        LS_LAUNCH_CHECK();
    }
    return run_filter_steps(lv, up_base, d_depth, height, width, filter->filter_strength,
                            filter->edge_threshold, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, d_keep, nullptr, 0, 0.0, st);
}

int ls_depth_filter_frame(const float *d_rgb, const float *d_depth, const uint8_t *d_alpha,
                          int64_t height, int64_t width, const ls_filter_params *filter,
                          float *d_frgb, float *d_fdepth, uint8_t *d_falpha, uint8_t *d_keep,
                          float *d_pyramid, void *stream) {
    if (!filter || !d_rgb || !d_depth || !d_alpha || !d_pyramid || height <= 0 || width <= 0)
        return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Levels lv{};
    float *up_base = nullptr;
    if (!setup_levels(height, width, filter->levels_n, d_pyramid, lv, up_base)) return LS_EINVAL;
    const int L = lv.L;
    k_to_sentinel_pool<<<grid_for(lv.h[1] * lv.w[1], 256), 256, 0, st>>>(d_depth, height, width,
                                                                         lv.img[0]);
    LS_LAUNCH_CHECK();
    for (int k = 2; k <= L; ++k) {
        k_min_pool<<<grid_for(lv.h[k] * lv.w[k], 256), 256, 0, st>>>(lv.img[k - 2], lv.h[k - 1],
                                                                     lv.w[k - 1], lv.img[k - 1]);
        LS_LAUNCH_CHECK();
    }
    return run_filter_steps(lv, up_base, d_depth, height, width, filter->filter_strength,
                            filter->edge_threshold, nullptr, d_rgb, d_alpha, d_frgb, d_fdepth,
                            d_falpha, d_keep, nullptr, 0, 0.0, st);
}

int64_t ls_filter_sweep_floats(int64_t height, int64_t width, int32_t levels_n,
                               int32_t n_strengths) {
    if (levels_n < 1 || levels_n > 5 || height <= 0 || width <= 0 || n_strengths < 1 ||
        n_strengths > kMaxSweep)
        return -1;
    int64_t h[9], w[9];
    level_sizes(height, width, levels_n, h, w);
    int64_t total = 0;
    for (int k = 1; k <= levels_n; ++k) total += h[k] * w[k];
    return total + (levels_n >= 2 ? (int64_t)n_strengths * h[1] * w[1] : 0);
}

int ls_depth_filter_sweep(const float *d_rgb, const float *d_depth, const uint8_t *d_alpha,
                          int64_t height, int64_t width, int32_t levels_n,
                          double edge_threshold, const double *h_strengths, int32_t n_strengths,
                          float *d_frgb, float *d_fdepth, uint8_t *d_falpha, uint8_t *d_keep,
                          float *d_work, void *stream) {
    if (!d_depth || !d_work || !h_strengths || height <= 0 || width <= 0 ||
        !(edge_threshold > 0.0) || n_strengths < 1 || n_strengths > kMaxSweep ||
        levels_n < 1 || levels_n > 5)
        return LS_EINVAL;
    if ((d_frgb || d_fdepth || d_falpha) && (!d_rgb || !d_alpha)) return LS_EINVAL;
    FsSweep sw{};
    for (int k = 0; k < n_strengths; ++k) {
        if (!(h_strengths[k] >= 0.0)) return LS_EINVAL;
        sw.fs[k] = h_strengths[k];
    }
    cudaStream_t st = (cudaStream_t)stream;
    Levels lv{};
    float *up_base = nullptr;
    if (!setup_levels(height, width, levels_n, d_work, lv, up_base)) return LS_EINVAL;
    const int L = lv.L;
    // strength-independent pyramid, once
    k_to_sentinel_pool<<<grid_for(lv.h[1] * lv.w[1], 256), 256, 0, st>>>(d_depth, height, width,
                                                                         lv.img[0]);
    LS_LAUNCH_CHECK();
    for (int k = 2; k <= L; ++k) {
        k_min_pool<<<grid_for(lv.h[k] * lv.w[k], 256), 256, 0, st>>>(lv.img[k - 2], lv.h[k - 1],
                                                                     lv.w[k - 1], lv.img[k - 1]);
        LS_LAUNCH_CHECK();
    }
    const float *coarse = lv.img[L - 1];
    int64_t cstride = 0;
    if (L >= 2) {  // every strength's non-final steps: one launch, z = strength
        sw.out_stride = lv.h[1] * lv.w[1];
        const dim3 g((unsigned)((lv.w[1] + kFuseTX - 1) / kFuseTX),
                     (unsigned)((lv.h[1] + kFuseTY - 1) / kFuseTY), (unsigned)n_strengths);
        cudaError_t e = launch_pdl(k_filter_coarse_fused<false>, g, dim3(256), 0, st, lv, up_base,
                                   sw, edge_threshold, FinalArgs{});
        if (e != cudaSuccess) return (int)e;
        coarse = up_base;
        cstride = sw.out_stride;
    }
    cudaError_t e = launch_pdl(k_filter_final_sweep, step_grid2(lv.h[1], lv.w[1]), dim3(32, 8),
                               0, st, coarse, cstride, lv.h[1], lv.w[1], d_depth, d_rgb, d_alpha,
                               height, width, sw, (int)n_strengths, edge_threshold, d_frgb,
                               d_fdepth, d_falpha, d_keep);
    return (int)e;
}

}  // extern "C"
