// U-Net convolutions on sm_100a tensor cores: implicit GEMM with TMA-fed
// operands, tcgen05.mma (kind::f16, bf16 x bf16 -> f32) with the accumulator in
// TMEM, and a fused epilogue (folded BatchNorm scale/shift, ReLU / leaky,
// 2x2 max pool, the final 1x1 conv + sigmoid, pixel-shuffle store of the 2x2
// transposed conv).
//
// GEMM view of one layer:  D[M = pixels][N = out channels] = A[M][K] * B[N][K]^T
//   A : im2col of the NHWC bf16 input, never materialised: TMA boxes of the
//       input whose out-of-bounds zero fill is the conv's "same" padding; the
//       decoder's [up, skip] concat is two tensor maps walked in K order.
//   B : the weights, K-major.
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

__device__ __forceinline__ float apply_act(float v, int act, float alpha) {
    if (act == LS_ACT_RELU) return v > 0.0f ? v : 0.0f;
    if (act == LS_ACT_LEAKY) return v > 0.0f ? v : alpha * v;
    return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

// ============================================================ conv kernel ==
// Persistent, warp-specialised implicit-GEMM convolution:
//   * 320 threads: warp 0 TMA producer, warp 1 MMA issuer, warps 2-9 epilogue
//     (two warps per TMEM lane quarter, splitting the column groups); one CTA
//     per SM loops over (pixel tile, column tile) work items.
//   * TMEM holds TWO accumulators (2 x BN columns): the epilogue drains tile i
//     while the MMA warp already accumulates tile i+1.
//   * Halo reuse: the pixel tile is 8 rows x 16 columns (m = row*16 + col) and
//     one TMA box of (8+2) rows x 16 columns per (kx, channel chunk) serves all
//     three ky taps -- tap ky is the same smem tile offset by ky*16 rows (two
//     whole 8-row swizzle atoms), so the descriptor start moves, not the data:
//     3 input loads per chunk instead of 9.
//   * Weights of small layers (<= kResidentMax bytes, one column tile) are
//     loaded into shared memory ONCE per CTA and stay resident; otherwise a
//     (kys x BN x chunk) weight box streams with every A box.
//   * Epilogue constants (folded-BN scale/shift, head weights) are staged in
//     shared memory once per CTA.
//   Weight layout: [tap][n][c] with tap = kx*kys + ky (kx-major).
constexpr int kTW = 16, kTH = 8;
constexpr size_t kResidentMax = 80 * 1024;
constexpr size_t kSmemBudget = 222 * 1024;

enum EpiMode { kPlain = 0, kPool = 1, kHead = 2, kTransposed = 3 };

struct ConvParamsP {
    int batch, h, w;
    int tiles_x, tiles_y, n_tiles_m, n_tiles_n, n_items;
    int c0, c1, ctot, nq0, nq;
    int kxs, kys, pad;
    int n_total, cout, act;
    float alpha;
    const float *scale, *shift;
    __nv_bfloat16 *y;
    float *y_f32;
    __nv_bfloat16 *pool;
    const float *head_w, *head_b;
    int head_c;
    float *head_out;
    int resident;          // weights resident in smem
    int stages;
    uint32_t a_bytes;      // A stage footprint (1024-aligned)
    uint32_t a_tx;         // TMA bytes of one A box
    uint32_t b_blk;        // bytes of one (kys x BN x chunk) weight block
    uint32_t off_b;        // resident weights
    uint32_t off_const;    // scale[n_total], shift[n_total], head_w, head_b (f32)
    uint32_t off_pool;     // pool / head staging
    uint32_t off_bar;      // barriers
    int dbg;               // experiments: bit0 skip MMA, bit1 skip stores, bit2 skip TMA A
    unsigned long long *dbg_ts;  // bit3: per-CTA event timestamps (globaltimer)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int BN, int CHUNK>
struct CfgP {
    static constexpr uint32_t kRow = CHUNK * 2;  // bytes per operand row
    static constexpr uint32_t kLayout =
        CHUNK == 64 ? kSwizzle128B : (CHUNK == 32 ? kSwizzle64B : kSwizzle32B);
    // epilogue warpgroups (4 warps = the 4 TMEM lane quarters) working on
    // different tiles concurrently, and TMEM accumulator buffers so the MMA
    // warp can run ahead of all of them
    static constexpr int kEpiGroups = BN >= 256 ? 1 : (BN >= 128 ? 2 : (BN >= 64 ? 3 : 4));
    static constexpr int kAcc = (512 / BN) < 2 * kEpiGroups ? (512 / BN) : 2 * kEpiGroups;
    static constexpr int kThreads = 64 + 128 * kEpiGroups;
    static constexpr int kTmemColsRaw = kAcc * BN;
    static constexpr int kTmemCols = kTmemColsRaw <= 32 ? 32 : (kTmemColsRaw <= 64 ? 64 :
                                     (kTmemColsRaw <= 128 ? 128 : (kTmemColsRaw <= 256 ? 256 : 512)));
    static constexpr int kGroups = BN / 16;
};

template <int BN, int CHUNK>
constexpr int threads_for() { return CfgP<BN, CHUNK>::kThreads; }

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint32_t hmax4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162 *>(&a);
    __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162 *>(&b);
    __nv_bfloat162 z = *reinterpret_cast<__nv_bfloat162 *>(&c);
    __nv_bfloat162 w = *reinterpret_cast<__nv_bfloat162 *>(&d);
    __nv_bfloat162 m = __hmax2(__hmax2(x, y), __hmax2(z, w));
    return *reinterpret_cast<uint32_t *>(&m);
}

template <int BN, int CHUNK, int MODE>
__global__ void __launch_bounds__(threads_for<BN, CHUNK>()) k_conv_p(const __grid_constant__ CUtensorMap mA0,
                                                         const __grid_constant__ CUtensorMap mA1,
                                                         const __grid_constant__ CUtensorMap mB,
                                                         const ConvParamsP p) {
    using C = CfgP<BN, CHUNK>;
    constexpr int KXS = MODE == kTransposed ? 1 : 3;
    constexpr int KYS = KXS;
    extern __shared__ uint8_t smem_raw[];
    // 1024-align inside the shared window (keeps the shared address space visible)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const int S = p.stages;
    const uint32_t stage_bytes = KXS * (p.a_bytes + (p.resident ? 0u : p.b_blk));
    float *sconst = reinterpret_cast<float *>(smem + p.off_const);
    const float *s_scale = sconst;
    const float *s_shift = sconst + p.n_total;
    const float *s_hw = sconst + 2 * p.n_total;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bar);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + C::kAcc;
    uint64_t *bres = tempty + C::kAcc;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bres + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, 1);
            }
            for (int a = 0; a < C::kAcc; ++a) {
                mbar_init(tfull + a, 1);
                mbar_init(tempty + a, 4);
            }
            mbar_init(bres, 1);
            fence_barrier_init();
            tma_prefetch(&mA0);
            if (p.c1 > 0) tma_prefetch(&mA1);
            tma_prefetch(&mB);
        }
        __syncwarp();
        tmem_alloc(tslot, C::kTmemCols);
    } else if (warp >= 2) {
        // stage the epilogue constants (visible after the __syncthreads below)
        const int t = threadIdx.x - 64;
        constexpr int kEpiThreads = 128 * C::kEpiGroups;
        for (int i = t; i < p.n_total; i += kEpiThreads) {
            sconst[i] = p.scale[i];
            sconst[p.n_total + i] = p.shift[i];
        }
        if (MODE == kHead)
            for (int i = t; i < p.head_c * p.cout; i += kEpiThreads)
                sconst[2 * p.n_total + i] = p.head_w[i];
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------ TMA producer ------------------------------
            if (p.resident) {
                mbar_expect_tx(bres, (uint32_t)(KXS * p.nq) * p.b_blk);
                for (int q = 0; q < p.nq; ++q)
                    for (int kx = 0; kx < KXS; ++kx) {
                        const bool second = q >= p.nq0;
                        const int kc = second ? p.c0 + (q - p.nq0) * CHUNK : q * CHUNK;
                        tma_load_3d(smem + p.off_b + (q * KXS + kx) * p.b_blk, &mB, kc, 0, kx * KYS,
                                    bres);
                    }
            }
            uint32_t it = 0;
            const int tpi = p.tiles_x * p.tiles_y;
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
                const int mt = item / p.n_tiles_n, nt = item - mt * p.n_tiles_n;
                const int img = mt / tpi, r = mt - img * tpi;
                const int y0 = (r / p.tiles_x) * kTH, x0 = (r % p.tiles_x) * kTW;
                const uint32_t tl = (uint32_t)((item - (int)blockIdx.x) / (int)gridDim.x);
                if ((p.dbg & 8) && !(p.dbg & 16) && tl < 64)
                    p.dbg_ts[(blockIdx.x * 4 + 2) * 64 + tl] = gtimer();
                // one stage = one channel chunk, all KXS input boxes (+ weight blocks)
                for (int q = 0; q < p.nq; ++q, ++it) {
                    const int s = (int)(it % (uint32_t)S);
                    const uint32_t ph = (it / (uint32_t)S) & 1u;
                    mbar_wait(empty + s, ph ^ 1u);
                    uint8_t *st = smem + (size_t)s * stage_bytes;
                    const bool second = q >= p.nq0;
                    const int c = (second ? q - p.nq0 : q) * CHUNK;
                    if (p.dbg & 4) {
                        mbar_arrive(full + s);
                        continue;
                    }
                    mbar_expect_tx(full + s, KXS * (p.a_tx + (p.resident ? 0u : p.b_blk)));
#pragma unroll
                    for (int kx = 0; kx < KXS; ++kx) {
                        tma_load_4d(st + kx * p.a_bytes, second ? &mA1 : &mA0, c, x0 + kx - p.pad,
                                    y0 - p.pad, img, full + s);
                        if (!p.resident)
                            tma_load_3d(st + KXS * p.a_bytes + kx * p.b_blk, &mB,
                                        (second ? p.c0 : 0) + c, nt * BN, kx * KYS, full + s);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------- MMA issuer -------------------------------
            // Descriptors are built once: per MMA only the 14-bit start-address
            // field (low word) moves, by compile-time offsets.
            const uint32_t idesc = idesc_bf16(128, BN);
            const uint64_t dproto = smem_desc(0, C::kRow, C::kLayout);
            const uint32_t dhi = (uint32_t)(dproto >> 32), dlo = (uint32_t)dproto;
            if (p.resident) mbar_wait(bres, 0);
            const uint32_t a_box16 = p.a_bytes >> 4, b_blk16 = p.b_blk >> 4;
            uint32_t it = 0, acc = 0;
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, ++acc) {
                const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
                if ((p.dbg & 8) && acc < 64) p.dbg_ts[(blockIdx.x * 4 + 0) * 64 + acc] = gtimer();
                mbar_wait(tempty + ab, aph ^ 1u);
                if ((p.dbg & 8) && acc < 64) p.dbg_ts[(blockIdx.x * 4 + 1) * 64 + acc] = gtimer();
                fence_after_sync();
                const uint32_t d = tmem + ab * BN;
                for (int q = 0; q < p.nq; ++q, ++it) {
                    const int s = (int)(it % (uint32_t)S);
                    const uint32_t ph = (it / (uint32_t)S) & 1u;
                    mbar_wait(full + s, ph);
                    if ((p.dbg & 16) && q == 0 && acc < 64)
                        p.dbg_ts[(blockIdx.x * 4 + 2) * 64 + acc] = gtimer();
                    fence_after_sync();
                    const uint32_t a_lo = dlo + ((sbase + (uint32_t)s * stage_bytes) >> 4);
                    const uint32_t b_lo =
                        dlo + ((p.resident ? sbase + p.off_b + (uint32_t)(q * KXS) * p.b_blk
                                           : sbase + (uint32_t)s * stage_bytes + KXS * p.a_bytes) >>
                               4);
                    if (!(p.dbg & 1)) {
#pragma unroll
                        for (int kx = 0; kx < KXS; ++kx) {
#pragma unroll
                            for (int ky = 0; ky < KYS; ++ky) {
#pragma unroll
                                for (int j = 0; j < CHUNK / 16; ++j) {
                                    const uint32_t ao = kx * a_box16 + (ky * kTW * C::kRow + 32 * j) / 16;
                                    const uint32_t bo = kx * b_blk16 + (ky * BN * C::kRow + 32 * j) / 16;
                                    const uint64_t adesc = ((uint64_t)dhi << 32) | (a_lo + ao);
                                    const uint64_t bdesc = ((uint64_t)dhi << 32) | (b_lo + bo);
                                    mma_bf16(d, adesc, bdesc, idesc,
                                             (q | kx | ky | j) != 0 ? 1u : 0u);
                                }
                            }
                        }
                    }
                    mma_commit(empty + s);
                    if ((p.dbg & 16) && q == 0 && acc < 64)
                        p.dbg_ts[(blockIdx.x * 4 + 3) * 64 + acc] = gtimer();
                }
                mma_commit(tfull + ab);
            }
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        // warpgroup eg (4 warps, one per TMEM lane quarter) drains every
        // kEpiGroups-th tile of this CTA, all column groups of it
        const int eg = (warp - 2) >> 2;
        const int quarter = warp & 3;            // TMEM lane quarter this warp may access
        const int m = quarter * 32 + lane;       // pixel row of the tile
        const int tx = m % kTW, ty = m / kTW;
        const uint32_t spool = sbase + p.off_pool + (uint32_t)eg * (128u * 32u);
        const int tpi = p.tiles_x * p.tiles_y;
        uint32_t acc = (uint32_t)eg;
        for (int item = blockIdx.x + eg * gridDim.x; item < p.n_items;
             item += C::kEpiGroups * gridDim.x, acc += C::kEpiGroups) {
            const int mt = item / p.n_tiles_n, nt = item - mt * p.n_tiles_n;
            const int img = mt / tpi, r = mt - img * tpi;
            const int gy = (r / p.tiles_x) * kTH + ty, gx = (r % p.tiles_x) * kTW + tx;
            const bool valid = gx < p.w && gy < p.h;
            const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
            mbar_wait(tfull + ab, aph);
            if ((p.dbg & 8) && !(p.dbg & 16) && acc < 64 && quarter == 0 && lane == 0)
                p.dbg_ts[(blockIdx.x * 4 + 3) * 64 + acc] = gtimer();
            fence_after_sync();
            const uint32_t trow = tmem + ab * BN + ((uint32_t)(quarter * 32) << 16);
            float hacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
            for (int g = 0; g < C::kGroups; ++g) {
                const int n = nt * BN + g * 16;
                if (n >= p.n_total) break;  // uniform
                uint32_t rr[16];
                tmem_ld16(trow + (uint32_t)(g * 16), rr);
                if (g + 1 == C::kGroups || n + 16 >= p.n_total) {
                    // accumulator fully read -> hand the TMEM buffer back early
                    fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty + ab);
                }
                float v[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    v[i] = apply_act(fmaf(__uint_as_float(rr[i]), s_scale[n + i], s_shift[n + i]),
                                     p.act, p.alpha);
                if (MODE == kHead) {
                    for (int j2 = 0; j2 < p.head_c; ++j2) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            hacc[j2] = fmaf(s_hw[j2 * p.cout + n + i], v[i], hacc[j2]);
                    }
                    if (!p.y && !p.y_f32) continue;  // head input not materialised
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
                if (valid && !(p.dbg & 2)) {
                    int64_t pix;
                    int o = n;
                    if (MODE == kTransposed) {
                        const int dd = n / p.cout;
                        o = n - dd * p.cout;
                        pix = ((int64_t)img * (2 * p.h) + 2 * gy + (dd >> 1)) * (2 * p.w) + 2 * gx +
                              (dd & 1);
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
                if (MODE == kPool) {
                    st_shared_v4(spool + m * 32, lo);
                    st_shared_v4(spool + m * 32 + 16, hi);
                    named_bar_sync(1 + eg, 128);
                    if (valid && !(tx & 1) && !(ty & 1)) {
                        uint4 o2[2];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const uint4 a0 = ld_shared_v4(spool + m * 32 + hh * 16);
                            const uint4 a1 = ld_shared_v4(spool + (m + 1) * 32 + hh * 16);
                            const uint4 a2 = ld_shared_v4(spool + (m + kTW) * 32 + hh * 16);
                            const uint4 a3 = ld_shared_v4(spool + (m + kTW + 1) * 32 + hh * 16);
                            o2[hh] = make_uint4(hmax4(a0.x, a1.x, a2.x, a3.x),
                                                hmax4(a0.y, a1.y, a2.y, a3.y),
                                                hmax4(a0.z, a1.z, a2.z, a3.z),
                                                hmax4(a0.w, a1.w, a2.w, a3.w));
                        }
                        const int64_t pp = ((int64_t)img * (p.h / 2) + gy / 2) * (p.w / 2) + gx / 2;
                        uint4 *dst = reinterpret_cast<uint4 *>(p.pool + pp * p.cout + n);
                        dst[0] = o2[0];
                        dst[1] = o2[1];
                    }
                    named_bar_sync(1 + eg, 128);
                }
            }
            if (MODE == kHead && valid) {
                const int64_t pix = ((int64_t)img * p.h + gy) * p.w + gx;
                for (int j2 = 0; j2 < p.head_c; ++j2) {
                    const float z = hacc[j2] + __ldg(p.head_b + j2);
                    p.head_out[pix * p.head_c + j2] = 1.0f / (1.0f + expf(-z));
                }
            }
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

}  // namespace unet
}  // namespace ls

using namespace ls::unet;

struct ls_conv_plan {
    CUtensorMap a0, a1, b;
    ConvParamsP p;
    int bn, chunk, grid, mode;
    size_t smem;
};

static bool chunk_ok(int c) { return c == 16 || c == 32 || (c > 0 && c % 64 == 0); }

namespace ls {
namespace unet {

static bool encode_act_p(CUtensorMap *map, const void *base, int c, int w, int h, int batch,
                         int chunk, int box_h) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
    cuuint32_t box[4] = {(cuuint32_t)chunk, (cuuint32_t)kTW, (cuuint32_t)box_h, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// weights [taps][n_total][ctot], box {chunk, bn, kys}
static bool encode_wts_p(CUtensorMap *map, const void *base, int ctot, int n_total, int taps,
                         int chunk, int bn, int kys) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)ctot, (cuuint64_t)n_total, (cuuint64_t)taps};
    cuuint64_t strides[2] = {(cuuint64_t)ctot * 2, (cuuint64_t)n_total * ctot * 2};
    cuuint32_t box[3] = {(cuuint32_t)chunk, (cuuint32_t)bn, (cuuint32_t)kys};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int CHUNK, int MODE>
static int launch_m(const ls_conv_plan *pl, cudaStream_t st) {
    static int attr_done = 0;  // idempotent: racing threads set the same value
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k_conv_p<BN, CHUNK, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(kSmemBudget + 2048));
        if (e != cudaSuccess) return (int)e;
        attr_done = 1;
    }
    k_conv_p<BN, CHUNK, MODE><<<pl->grid, CfgP<BN, CHUNK>::kThreads, pl->smem, st>>>(
        pl->a0, pl->a1, pl->b, pl->p);
    return (int)cudaGetLastError();
}

template <int BN, int CHUNK>
static int launch_p(const ls_conv_plan *pl, cudaStream_t st) {
    switch (pl->mode) {
        case kPlain: return launch_m<BN, CHUNK, kPlain>(pl, st);
        case kPool: return launch_m<BN, CHUNK, kPool>(pl, st);
        case kHead: return launch_m<BN, CHUNK, kHead>(pl, st);
        default: return launch_m<BN, CHUNK, kTransposed>(pl, st);
    }
}

}  // namespace unet
}  // namespace ls

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
    if (!d_x0 || !d_w || !d_scale || !d_shift || batch < 1 || h < 1 || w < 1 || !chunk_ok(c0))
        return fail(LS_EINVAL);
    if (c1 < 0 || (c1 > 0 && (!d_x1 || !chunk_ok(c1)))) return fail(LS_EINVAL);
    if (cout < 16 || cout % 16 || (ksize != 1 && ksize != 3)) return fail(LS_EINVAL);
    if (transposed && (ksize != 1 || c1 != 0 || d_pool || d_head_w)) return fail(LS_EINVAL);
    if (d_pool && (h % 2 || w % 2)) return fail(LS_EINVAL);
    if (d_head_w && (head_c < 1 || head_c > 4 || !d_head_b || !d_head_out)) return fail(LS_EINVAL);
    const int n_total = transposed ? 4 * cout : cout;
    if (n_total > 4096) return fail(LS_EINVAL);
    int bn = n_total >= 256 ? 256 : (n_total >= 128 ? 128 : (n_total >= 64 ? 64 : 32));
    if (n_total % bn) bn = 32;
    if (d_head_w && n_total > bn) return fail(LS_EINVAL);  // the head needs every channel
    int chunk = bn >= 256 ? 32 : 64;
    while (chunk > 16 && ((c0 % chunk) || (c1 % chunk))) chunk >>= 1;

    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan;
    if (!pl) return fail(LS_EINVAL);
    ConvParamsP &p = pl->p;
    p.batch = batch;
    p.h = h;
    p.w = w;
    p.tiles_x = (w + kTW - 1) / kTW;
    p.tiles_y = (h + kTH - 1) / kTH;
    p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
    p.c0 = c0;
    p.c1 = c1;
    p.ctot = c0 + c1;
    p.kxs = ksize == 3 ? 3 : 1;
    p.kys = ksize == 3 ? 3 : 1;
    p.pad = ksize == 3 ? 1 : 0;
    p.n_total = n_total;
    p.cout = cout;
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
    const char *env_st = getenv("LS_CONV_MAX_STAGES");  // tuning experiments only
    const int max_stages = env_st ? atoi(env_st) : 8;
    const int box_h = kTH + 2 * p.pad;
    const size_t const_bytes = ((size_t)(2 * n_total + (d_head_w ? head_c * cout : 0)) * 4 + 1023) &
                               ~size_t(1023);
    size_t res_bytes = 0, stage_bytes = 0;
    int stages = 0;
    // shrink the K chunk, then the column tile, until >= 2 pipeline stages fit
    for (;;) {
        const uint32_t row = (uint32_t)chunk * 2;
        p.nq0 = c0 / chunk;
        p.nq = (c0 + c1) / chunk;
        p.a_tx = (uint32_t)(kTW * box_h) * row;
        p.a_bytes = (p.a_tx + 1023u) & ~1023u;
        p.n_tiles_n = (n_total + bn - 1) / bn;
        p.n_items = p.n_tiles_m * p.n_tiles_n;
        p.b_blk = (uint32_t)(p.kys * bn) * row;
        const size_t nk = (size_t)p.kxs * p.nq;
        p.resident = (p.n_tiles_n == 1 && nk * p.b_blk <= kResidentMax) ? 1 : 0;
        res_bytes = p.resident ? nk * p.b_blk : 0;
        stage_bytes = (size_t)p.kxs * (p.a_bytes + (p.resident ? 0 : p.b_blk));
        const size_t fixed = res_bytes + const_bytes + 16384 + 512;
        stages = kSmemBudget > fixed ? (int)((kSmemBudget - fixed) / stage_bytes) : 0;
        if (stages >= 2) break;
        if (chunk > 16 && (c0 % (chunk / 2)) == 0 && (c1 % (chunk / 2)) == 0) {
            chunk >>= 1;
        } else if (bn > 32 && !d_head_w) {
            bn >>= 1;
        } else {
            delete pl;
            return fail(LS_EINVAL);
        }
    }
    if (stages > max_stages) stages = max_stages;
    p.stages = stages;
    p.off_b = (uint32_t)(stages * stage_bytes);
    p.off_const = (uint32_t)(p.off_b + res_bytes);
    p.off_pool = (uint32_t)(p.off_const + const_bytes);
    p.off_bar = p.off_pool + 16384;
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = bn;
    pl->chunk = chunk;
    pl->mode = transposed ? kTransposed : (d_head_w ? kHead : (d_pool ? kPool : kPlain));
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    const char *env_dbg = getenv("LS_CONV_DBG");
    p.dbg = env_dbg ? atoi(env_dbg) : 0;
    p.dbg_ts = nullptr;
    if (p.dbg & 8) cudaMalloc(&p.dbg_ts, 148 * 4 * 64 * sizeof(unsigned long long));
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    bool ok = encode_act_p(&pl->a0, d_x0, c0, w, h, batch, chunk, box_h);
    ok = ok && encode_act_p(&pl->a1, c1 > 0 ? d_x1 : d_x0, c1 > 0 ? c1 : c0, w, h, batch, chunk,
                            box_h);
    ok = ok && encode_wts_p(&pl->b, d_w, p.ctot, n_total, p.kxs * p.kys, chunk, bn, p.kys);
    if (!ok) {
        delete pl;
        return fail(LS_EINVAL);
    }
    if (status) *status = 0;
    return pl;
}

int ls_conv_plan_launch(const ls_conv_plan *pl, void *stream) {
    if (!pl) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
#define LS_CASE(B, K) \
    if (pl->bn == B && pl->chunk == K) return launch_p<B, K>(pl, st);
    LS_CASE(32, 16) LS_CASE(32, 32) LS_CASE(32, 64)
    LS_CASE(64, 16) LS_CASE(64, 32) LS_CASE(64, 64)
    LS_CASE(128, 16) LS_CASE(128, 32) LS_CASE(128, 64)
    LS_CASE(256, 16) LS_CASE(256, 32)
#undef LS_CASE
    return LS_EINVAL;
}

void ls_conv_plan_destroy(ls_conv_plan *pl) {
    if (pl && pl->p.dbg_ts) cudaFree(pl->p.dbg_ts);
    delete pl;
}

/* experiments only: copy the per-CTA event timestamps (LS_CONV_DBG bit 3) */
int ls_conv_plan_debug_ts(const ls_conv_plan *pl, unsigned long long *host, int n) {
    if (!pl || !pl->p.dbg_ts || n > 148 * 4 * 64) return LS_EINVAL;
    return (int)cudaMemcpy(host, pl->p.dbg_ts, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}

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
