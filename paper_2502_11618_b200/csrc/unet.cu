// U-Net convolutions on sm_100a tensor cores: implicit GEMM with TMA-fed
// operands, tcgen05.mma (kind::f16, bf16 x bf16 -> f32) and the accumulator in
// TMEM, plus a fused epilogue (folded BatchNorm scale/shift, ReLU / leaky,
// 2x2 max pool, the final 1x1 conv + sigmoid, pixel-shuffle store of the
// 2x2 transposed conv).
//
// GEMM view of one layer:  D[M = pixels][N = out channels] = A[M][K] * B[N][K]^T
//   A  : im2col of the NHWC bf16 input, never materialised -- for every K chunk
//        (tap ky,kx x channel chunk) one 4-D TMA box {chunk, TW, TH, 1} of the
//        input at (c, x0+kx-1, y0+ky-1, n); TMA's out-of-bounds zero fill is
//        the conv's zero "same" padding.  The decoder's [up, skip] concat is
//        two tensor maps walked in K order, never copied.
//   B  : the weights, K-major [N][taps*C], one 2-D TMA box {chunk, BN}.
// CTA = 128 threads, one 128-pixel tile (TH rows x TW cols) x BN columns:
//   warp 0 lane 0 : TMA producer over a STAGES-deep smem ring (mbarriers)
//   warp 1 lane 0 : tcgen05.mma issuer, 128 x BN x 16 per instruction,
//                   tcgen05.commit frees each stage and finally signals TMEM full
//   warps 0-3     : epilogue, warp w reads TMEM lanes 32w..32w+31 (its pixels)
// Two CTAs fit one SM (<= ~100 KB smem, <= 256 TMEM columns each), so one
// CTA's epilogue overlaps the other's main loop.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include <new>

#include "lidarsplat_cuda.h"
#include "lidarsplat_unet.h"
#include "umma.cuh"

namespace ls {
namespace unet {

using namespace ls::umma;

struct ConvParams {
    int batch, h, w;        // input spatial dims
    int tw, th;             // pixel tile = th rows x tw cols (tw*th = 128)
    int tiles_x, tiles_y;   // tiles per image
    int c0, c1, ctot;       // source channels
    int chunk;              // K chunk width in channels (16 / 32 / 64)
    int nq0, nq;            // chunks from source 0 / per tap in total
    int taps, pad;          // 9,1 (3x3) or 1,0
    int n_total;            // GEMM N (cout, or 4*cout transposed)
    int cout;               // channels of one output pixel
    int transposed;
    int act;
    float alpha;
    const float *scale, *shift;
    __nv_bfloat16 *y;
    float *y_f32;
    __nv_bfloat16 *pool;
    const float *head_w, *head_b;
    int head_c;
    float *head_out;
    uint32_t swz_layout, row_bytes;
};

constexpr int kThreads = 128;
constexpr int kTileM = 128;
constexpr int kMaxRowBytes = 128;  // chunk <= 64 bf16

template <int BN>
struct Cfg {
    static constexpr int kStages = BN <= 32 ? 5 : (BN <= 64 ? 4 : (BN <= 128 ? 3 : 2));
    static constexpr int kABytes = kTileM * kMaxRowBytes;
    static constexpr int kBBytes = BN * kMaxRowBytes;
    static constexpr int kTmemCols = BN < 32 ? 32 : BN;
    static constexpr size_t kSmem =
        1024 + (size_t)kStages * (kABytes + kBBytes) + (2 * kStages + 1) * 8 + 16;
};

__device__ __forceinline__ float apply_act(float v, int act, float alpha) {
    if (act == LS_ACT_RELU) return v > 0.0f ? v : 0.0f;
    if (act == LS_ACT_LEAKY) return v > 0.0f ? v : alpha * v;
    return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

template <int BN>
__global__ void __launch_bounds__(kThreads) k_conv(const __grid_constant__ CUtensorMap mA0,
                                                   const __grid_constant__ CUtensorMap mA1,
                                                   const __grid_constant__ CUtensorMap mB,
                                                   const ConvParams p) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = sA + C::kStages * C::kABytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + C::kStages * C::kBBytes);
    uint64_t *empty = full + C::kStages;
    uint64_t *accf = empty + C::kStages;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(accf + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_img = p.tiles_x * p.tiles_y;
    const int img = blockIdx.x / tiles_img;
    const int rem = blockIdx.x - img * tiles_img;
    const int y0 = (rem / p.tiles_x) * p.th;
    const int x0 = (rem % p.tiles_x) * p.tw;
    const int n0 = blockIdx.y * BN;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < C::kStages; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, 1);
            }
            mbar_init(accf, 1);
            fence_barrier_init();
            tma_prefetch(&mA0);
            if (p.c1 > 0) tma_prefetch(&mA1);
            tma_prefetch(&mB);
        }
        __syncwarp();
        tmem_alloc(tslot, C::kTmemCols);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;

    const int nk = p.taps * p.nq;
    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        const uint32_t tx_bytes = (uint32_t)(kTileM + BN) * p.row_bytes;
        for (int kk = 0; kk < nk; ++kk) {
            const int s = kk % C::kStages;
            const uint32_t ph = (uint32_t)(kk / C::kStages) & 1u;
            mbar_wait(empty + s, ph ^ 1u);
            const int tap = kk / p.nq, q = kk - tap * p.nq;
            const int ky = p.taps == 9 ? tap / 3 : 0, kx = p.taps == 9 ? tap % 3 : 0;
            const bool second = q >= p.nq0;
            const int c = (second ? q - p.nq0 : q) * p.chunk;
            const int kb = tap * p.ctot + (second ? p.c0 : 0) + c;
            mbar_expect_tx(full + s, tx_bytes);
            tma_load_4d(sA + s * C::kABytes, second ? &mA1 : &mA0, c, x0 + kx - p.pad,
                        y0 + ky - p.pad, img, full + s);
            tma_load_2d(sB + s * C::kBBytes, &mB, kb, n0, full + s);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = idesc_bf16(kTileM, BN);
        const int ksteps = p.chunk / 16;
        for (int kk = 0; kk < nk; ++kk) {
            const int s = kk % C::kStages;
            const uint32_t ph = (uint32_t)(kk / C::kStages) & 1u;
            mbar_wait(full + s, ph);
            fence_after_sync();
            const uint32_t a0 = smem_u32(sA + s * C::kABytes);
            const uint32_t b0 = smem_u32(sB + s * C::kBBytes);
            for (int j = 0; j < ksteps; ++j) {
                mma_bf16(tmem, smem_desc(a0 + 32u * j, p.row_bytes, p.swz_layout),
                         smem_desc(b0 + 32u * j, p.row_bytes, p.swz_layout), idesc,
                         (kk | j) != 0 ? 1u : 0u);
            }
            mma_commit(empty + s);
        }
        mma_commit(accf);
    }
    __syncwarp();

    // ---------------- epilogue ----------------
    mbar_wait(accf, 0);
    fence_after_sync();
    const int m = warp * 32 + lane;
    const int tx = m % p.tw, ty = m / p.tw;
    const int gx = x0 + tx, gy = y0 + ty;
    const bool valid = gx < p.w && gy < p.h;
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    float hacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    __nv_bfloat16 *stage = reinterpret_cast<__nv_bfloat16 *>(sA);  // pipeline drained
#pragma unroll 1
    for (int g = 0; g < BN / 16; ++g) {
        const int n = n0 + g * 16;
        if (n >= p.n_total) break;  // warp-uniform
        uint32_t r[16];
        tmem_ld16(trow + (uint32_t)(g * 16), r);
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float a = __uint_as_float(r[i]);
            const float sc = p.scale ? __ldg(p.scale + n + i) : 1.0f;
            const float sh = p.shift ? __ldg(p.shift + n + i) : 0.0f;
            v[i] = apply_act(fmaf(a, sc, sh), p.act, p.alpha);
        }
        if (p.head_w) {
            for (int j = 0; j < p.head_c; ++j) {
#pragma unroll
                for (int i = 0; i < 16; ++i) hacc[j] = fmaf(__ldg(p.head_w + j * p.cout + n + i), v[i], hacc[j]);
            }
        }
        uint4 lo, hi;
        lo.x = pack_bf16(v[0], v[1]);
        lo.y = pack_bf16(v[2], v[3]);
        lo.z = pack_bf16(v[4], v[5]);
        lo.w = pack_bf16(v[6], v[7]);
        hi.x = pack_bf16(v[8], v[9]);
        hi.y = pack_bf16(v[10], v[11]);
        hi.z = pack_bf16(v[12], v[13]);
        hi.w = pack_bf16(v[14], v[15]);
        if (valid) {
            int64_t pix;
            int o = n;
            if (p.transposed) {
                const int d = n / p.cout;
                o = n - d * p.cout;
                pix = ((int64_t)img * (2 * p.h) + 2 * gy + (d >> 1)) * (2 * p.w) + 2 * gx + (d & 1);
            } else {
                pix = ((int64_t)img * p.h + gy) * p.w + gx;
            }
            if (p.y) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.y + pix * p.cout + o);
                dst[0] = lo;
                dst[1] = hi;
            }
            if (p.y_f32) {
                float4 *dst = reinterpret_cast<float4 *>(p.y_f32 + pix * p.cout + o);
                dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                dst[2] = make_float4(v[8], v[9], v[10], v[11]);
                dst[3] = make_float4(v[12], v[13], v[14], v[15]);
            }
        }
        if (p.pool) {
            uint4 *srow = reinterpret_cast<uint4 *>(stage + m * 16);
            srow[0] = lo;
            srow[1] = hi;
            __syncthreads();
            if (valid && !(tx & 1) && !(ty & 1)) {
                const __nv_bfloat162 *r0 = reinterpret_cast<const __nv_bfloat162 *>(stage + m * 16);
                const __nv_bfloat162 *r1 = reinterpret_cast<const __nv_bfloat162 *>(stage + (m + 1) * 16);
                const __nv_bfloat162 *r2 = reinterpret_cast<const __nv_bfloat162 *>(stage + (m + p.tw) * 16);
                const __nv_bfloat162 *r3 = reinterpret_cast<const __nv_bfloat162 *>(stage + (m + p.tw + 1) * 16);
                uint32_t outw[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    __nv_bfloat162 mx = __hmax2(__hmax2(r0[i], r1[i]), __hmax2(r2[i], r3[i]));
                    outw[i] = *reinterpret_cast<uint32_t *>(&mx);
                }
                const int64_t pp = ((int64_t)img * (p.h / 2) + gy / 2) * (p.w / 2) + gx / 2;
                uint4 *dst = reinterpret_cast<uint4 *>(p.pool + pp * p.cout + n);
                dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
                dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
            }
            __syncthreads();
        }
    }
    if (p.head_w && valid) {
        const int64_t pix = ((int64_t)img * p.h + gy) * p.w + gx;
        for (int j = 0; j < p.head_c; ++j) {
            const float z = hacc[j] + __ldg(p.head_b + j);
            p.head_out[pix * p.head_c + j] = 1.0f / (1.0f + expf(-z));
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
}

// ------------------------------------------------------------------ host ---

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

static CUtensorMapSwizzle swizzle_for(int row_bytes) {
    return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

static bool encode_act(CUtensorMap *map, const void *base, int c, int w, int h, int batch,
                       int chunk, int tw, int th) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
    cuuint32_t box[4] = {(cuuint32_t)chunk, (cuuint32_t)tw, (cuuint32_t)th, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool encode_wts(CUtensorMap *map, const void *base, int k_total, int n_total, int chunk,
                       int bn) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)k_total, (cuuint64_t)n_total};
    cuuint64_t strides[1] = {(cuuint64_t)k_total * 2};
    cuuint32_t box[2] = {(cuuint32_t)chunk, (cuuint32_t)bn};
    cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static int launch_bn(const CUtensorMap &a0, const CUtensorMap &a1, const CUtensorMap &b,
                     const ConvParams &p, dim3 grid, cudaStream_t st) {
    static bool attr_done = false;  // idempotent; racing threads set the same value
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k_conv<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)Cfg<BN>::kSmem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    k_conv<BN><<<grid, kThreads, Cfg<BN>::kSmem, st>>>(a0, a1, b, p);
    return (int)cudaGetLastError();
}

}  // namespace unet
}  // namespace ls

using namespace ls::unet;

struct ls_conv_plan {
    CUtensorMap a0, a1, b;
    ConvParams p;
    dim3 grid;
    int bn;
};

static bool chunk_ok(int c) { return c == 16 || c == 32 || (c > 0 && c % 64 == 0); }

extern "C" {

ls_conv_plan *ls_conv_plan_create(const uint16_t *d_x0, int32_t c0, const uint16_t *d_x1,
                                  int32_t c1, int32_t batch, int32_t h, int32_t w,
                                  const uint16_t *d_w, int32_t ksize, int32_t cout,
                                  int32_t transposed, const float *d_scale, const float *d_shift,
                                  int32_t act, float alpha, uint16_t *d_y, float *d_y_f32,
                                  uint16_t *d_pool, const float *d_head_w, const float *d_head_b,
                                  int32_t head_c, float *d_head_out, int32_t *status) {
    auto fail = [&](int rc) -> ls_conv_plan * {
        if (status) *status = rc;
        return nullptr;
    };
    if (!d_x0 || !d_w || batch < 1 || h < 1 || w < 1 || !chunk_ok(c0)) return fail(LS_EINVAL);
    if (c1 < 0 || (c1 > 0 && (!d_x1 || !chunk_ok(c1)))) return fail(LS_EINVAL);
    if (cout < 16 || cout % 16 || (ksize != 1 && ksize != 3)) return fail(LS_EINVAL);
    if (transposed && (ksize != 1 || c1 != 0 || d_pool || d_head_w)) return fail(LS_EINVAL);
    if (d_pool && (h % 2 || w % 2)) return fail(LS_EINVAL);
    if (d_head_w && (head_c < 1 || head_c > 4 || !d_head_b || !d_head_out)) return fail(LS_EINVAL);
    // chunk: widest of 64/32/16 channels dividing both sources
    int chunk = 64;
    while (chunk > 16 && ((c0 % chunk) || (c1 % chunk))) chunk >>= 1;
    const int n_total = transposed ? 4 * cout : cout;
    if (n_total > 4096) return fail(LS_EINVAL);
    int bn = n_total >= 256 ? 256 : (n_total >= 128 ? 128 : (n_total >= 64 ? 64 : 32));
    if (n_total % bn) bn = 32;
    if (d_head_w && n_total > bn) return fail(LS_EINVAL);  // the head needs every channel in one CTA
    int tw = 64;
    while (tw > 8 && (w % tw)) tw >>= 1;
    if (tw > w) tw = 8;
    const int th = 128 / tw;

    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan;
    if (!pl) return fail(LS_EINVAL);
    ConvParams &p = pl->p;
    p.batch = batch;
    p.h = h;
    p.w = w;
    p.tw = tw;
    p.th = th;
    p.tiles_x = (w + tw - 1) / tw;
    p.tiles_y = (h + th - 1) / th;
    p.c0 = c0;
    p.c1 = c1;
    p.ctot = c0 + c1;
    p.chunk = chunk;
    p.nq0 = c0 / chunk;
    p.nq = (c0 + c1) / chunk;
    p.taps = ksize == 3 ? 9 : 1;
    p.pad = ksize == 3 ? 1 : 0;
    p.n_total = n_total;
    p.cout = cout;
    p.transposed = transposed ? 1 : 0;
    p.act = act;
    p.alpha = alpha;
    p.scale = d_scale;
    p.shift = d_shift;
    p.y = reinterpret_cast<__nv_bfloat16 *>(d_y);
    p.y_f32 = d_y_f32;
    p.pool = reinterpret_cast<__nv_bfloat16 *>(d_pool);
    p.head_w = d_head_w;
    p.head_b = d_head_b;
    p.head_c = head_c;
    p.head_out = d_head_out;
    p.row_bytes = (uint32_t)chunk * 2;
    p.swz_layout = chunk == 64 ? kSwizzle128B : (chunk == 32 ? kSwizzle64B : kSwizzle32B);
    bool ok = encode_act(&pl->a0, d_x0, c0, w, h, batch, chunk, tw, th);
    ok = ok && encode_act(&pl->a1, c1 > 0 ? d_x1 : d_x0, c1 > 0 ? c1 : c0, w, h, batch, chunk, tw, th);
    ok = ok && encode_wts(&pl->b, d_w, p.taps * p.ctot, n_total, chunk, bn);
    if (!ok) {
        delete pl;
        return fail(LS_EINVAL);
    }
    pl->grid = dim3((unsigned)(p.tiles_x * p.tiles_y * batch), (unsigned)((n_total + bn - 1) / bn));
    pl->bn = bn;
    if (status) *status = 0;
    return pl;
}

int ls_conv_plan_launch(const ls_conv_plan *pl, void *stream) {
    if (!pl) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    switch (pl->bn) {
        case 32: return launch_bn<32>(pl->a0, pl->a1, pl->b, pl->p, pl->grid, st);
        case 64: return launch_bn<64>(pl->a0, pl->a1, pl->b, pl->p, pl->grid, st);
        case 128: return launch_bn<128>(pl->a0, pl->a1, pl->b, pl->p, pl->grid, st);
        case 256: return launch_bn<256>(pl->a0, pl->a1, pl->b, pl->p, pl->grid, st);
        default: return LS_EINVAL;
    }
}

void ls_conv_plan_destroy(ls_conv_plan *pl) { delete pl; }

int ls_conv2d(const uint16_t *d_x0, int32_t c0, const uint16_t *d_x1, int32_t c1, int32_t batch,
              int32_t h, int32_t w, const uint16_t *d_w, int32_t ksize, int32_t cout,
              const float *d_scale, const float *d_shift, int32_t act, float alpha,
              uint16_t *d_y, float *d_y_f32, uint16_t *d_pool, const float *d_head_w,
              const float *d_head_b, int32_t head_c, float *d_head_out, void *stream) {
    int32_t rc = 0;
    ls_conv_plan *pl = ls_conv_plan_create(d_x0, c0, d_x1, c1, batch, h, w, d_w, ksize, cout, 0,
                                           d_scale, d_shift, act, alpha, d_y, d_y_f32, d_pool,
                                           d_head_w, d_head_b, head_c, d_head_out, &rc);
    if (!pl) return rc;
    rc = ls_conv_plan_launch(pl, stream);
    ls_conv_plan_destroy(pl);
    return rc;
}

int ls_conv_transpose2x2(const uint16_t *d_x, int32_t cin, int32_t batch, int32_t h, int32_t w,
                         const uint16_t *d_w, int32_t cout, const float *d_scale,
                         const float *d_shift, uint16_t *d_y, void *stream) {
    int32_t rc = 0;
    ls_conv_plan *pl = ls_conv_plan_create(d_x, cin, nullptr, 0, batch, h, w, d_w, 1, cout, 1,
                                           d_scale, d_shift, LS_ACT_NONE, 0.0f, d_y, nullptr,
                                           nullptr, nullptr, nullptr, 0, nullptr, &rc);
    if (!pl) return rc;
    rc = ls_conv_plan_launch(pl, stream);
    ls_conv_plan_destroy(pl);
    return rc;
}

}  // extern "C"
