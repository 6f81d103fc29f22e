// U-Net convolutions on sm_100a tensor cores: implicit GEMM with TMA-fed
// operands, tcgen05.mma (kind::f16, bf16 x bf16 -> f32) with the accumulators
// in TMEM, and a fused epilogue (folded BatchNorm scale/shift, ReLU / leaky,
// 2x2 max pool, the final 1x1 conv + sigmoid, pixel-shuffle store of the 2x2
// transposed conv).
//
// GEMM view of one layer:  D[M = pixels][N = out channels] = A[M][K] * B[N][K]^T
//   A : im2col of the NHWC bf16 input, never materialised; the decoder's
//       [up, skip] concat is two tensor maps walked in K order.
//   B : the weights, K-major, layout [tap][n][c] with tap = kx*3 + ky.
//
// Halo tiles with a padded row pitch.  A work item is R image rows x 16
// columns.  For every channel chunk ONE TMA box of (R+2) rows x 18 columns of
// the input (TMA's out-of-bounds zero fill = the conv's zero padding) lands in
// shared memory as a K-major swizzled tile whose smem row r is the input pixel
// (r / 18, r % 18) of the halo window.  The GEMM rows use the same indexing
// (output pixel (r / 18, r % 18); columns 16 and 17 are junk and discarded), so
// tap (ky, kx) is just the descriptor start moved by ky*18 + kx rows -- all 9
// taps read one box.  This relies on the tensor core applying the swizzle on
// absolute shared-memory address bits (measured: scripts/umma_shift_test.cu --
// every row shift 0..8 is exact with base_offset 0, for 32/64/128 B swizzle).
// R = 7*MT rows, so the item is MT blocks of 128 GEMM rows (126 used).
// The 2x2 transposed conv has no halo: pitch 16, R = 8*MT, one tap.
//
// Kernel structure (persistent, warp-specialised, one CTA per SM):
//   warp 0 lane 0 : TMA producer over a STAGES-deep shared-memory ring
//   warp 1 lane 0 : tcgen05.mma issuer (descriptors precomputed: per MMA only
//                   the 14-bit start-address field moves)
//   warps 2..     : kEpiGroups epilogue warpgroups, each draining a different
//                   work item (4 warps = the 4 TMEM lane quarters)
// TMEM holds kAcc items' worth of accumulators, so the MMA warp runs ahead.
// Small weight tensors (<= kResidentMax, one column tile) stay resident in
// shared memory for the whole CTA; otherwise weight boxes stream with A.
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

constexpr int kTW = 16;  // output columns per item
constexpr size_t kResidentMax = 80 * 1024;
constexpr size_t kSmemBudget = 222 * 1024;

enum EpiMode { kPlain = 0, kPool = 1, kHead = 2, kTransposed = 3 };

struct ConvParamsP {
    int batch, h, w;
    int tiles_x, tiles_y, n_tiles_m, n_tiles_n, n_items;
    int c0, c1, ctot, nq0, nq;
    int kxps;               // kx taps per pipeline stage (1 or 3; 1 for transposed)
    int n_total, cout, act;
    float alpha;
    const float *scale, *shift;
    __nv_bfloat16 *y;
    float *y_f32;
    __nv_bfloat16 *pool;
    const float *head_w, *head_b;
    int head_c;
    float *head_out;
    int resident;           // weights resident in smem
    int stages;
    uint32_t a_bytes;       // A box footprint (1024-aligned)
    uint32_t a_tx;          // TMA bytes of one A box
    uint32_t b_tap;         // bytes of one tap's (BN x chunk) weight block
    uint32_t stage_bytes;
    uint32_t off_b;         // resident weights
    uint32_t off_const;     // scale[n_total], shift[n_total], head_w (f32)
    uint32_t off_stage;     // pool staging (per epilogue group)
    uint32_t stage_grp;     // bytes of one group's pool staging
    uint32_t off_bar;       // barriers
};

template <int BN, int CHUNK, int MODE>
struct CfgP {
    static constexpr uint32_t kRow = CHUNK * 2;  // bytes per operand row
    static constexpr uint32_t kLayout =
        CHUNK == 64 ? kSwizzle128B : (CHUNK == 32 ? kSwizzle64B : kSwizzle32B);
    static constexpr bool kConv3 = MODE != kTransposed;
    static constexpr int kTaps = kConv3 ? 9 : 1;
    static constexpr int kKys = kConv3 ? 3 : 1;
    static constexpr int kPitch = kConv3 ? 18 : 16;              // smem rows per image row
    static constexpr int kMT = BN <= 32 ? 4 : (BN <= 64 ? 2 : 1);  // 128-row blocks per item
    // image rows per item (even when pooling so 2x2 windows never straddle items)
    static constexpr int kR = kConv3 ? ((MODE == kPool && (7 * kMT) % 2) ? 7 * kMT - 1 : 7 * kMT)
                                     : 8 * kMT;
    static constexpr int kItemCols = kMT * BN;                   // TMEM columns per item
    static constexpr int kAcc = 512 / kItemCols >= 4 ? 4 : 512 / kItemCols;
    static constexpr int kEpiGroups = kAcc >= 4 ? 3 : (kAcc >= 3 ? 2 : 1);
    static constexpr int kThreads = 64 + 128 * kEpiGroups;
    static constexpr int kTmemCols = kAcc * kItemCols <= 32 ? 32 :
                                     (kAcc * kItemCols <= 64 ? 64 :
                                     (kAcc * kItemCols <= 128 ? 128 :
                                     (kAcc * kItemCols <= 256 ? 256 : 512)));
};

template <int BN, int CHUNK, int MODE>
constexpr int threads_for() { return CfgP<BN, CHUNK, MODE>::kThreads; }

__device__ __forceinline__ float apply_act(float v, int act, float alpha) {
    if (act == LS_ACT_RELU) return v > 0.0f ? v : 0.0f;
    if (act == LS_ACT_LEAKY) return v > 0.0f ? v : alpha * v;
    return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

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

// floor(a / b) for 0 <= a < 2^24, b >= 1 via one f32 reciprocal + correction
// (the lone producer / MMA threads are latency-bound; int32 division is ~30
// dependent instructions).
__device__ __forceinline__ int fdiv(int a, int b, float rb) {
    int q = (int)((float)a * rb);
    q -= (q * b > a);
    q += ((q + 1) * b <= a);
    return q;
}

struct ItemPos {
    int img, y0, x0, nt;
};

__device__ __forceinline__ ItemPos item_pos(const ConvParamsP &p, int item, float r_nt, float r_tpi,
                                            float r_tx, int rows) {
    ItemPos ip;
    const int mt = fdiv(item, p.n_tiles_n, r_nt);
    ip.nt = item - mt * p.n_tiles_n;
    const int tpi = p.tiles_x * p.tiles_y;
    ip.img = fdiv(mt, tpi, r_tpi);
    const int r = mt - ip.img * tpi;
    const int ty = fdiv(r, p.tiles_x, r_tx);
    ip.y0 = ty * rows;
    ip.x0 = (r - ty * p.tiles_x) * kTW;
    return ip;
}

template <int BN, int CHUNK, int MODE>
__global__ void __launch_bounds__(threads_for<BN, CHUNK, MODE>()) k_conv_p(
    const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
    const __grid_constant__ CUtensorMap mB, const ConvParamsP p) {
    using C = CfgP<BN, CHUNK, MODE>;
    constexpr int MT = C::kMT, KYS = C::kKys, P = C::kPitch, R = C::kR;
    extern __shared__ uint8_t smem_raw[];
    // 1024-align inside the shared window (keeps the shared address space visible)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const int S = p.stages;
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
    const float r_nt = 1.0f / (float)p.n_tiles_n;
    const float r_tpi = 1.0f / (float)(p.tiles_x * p.tiles_y);
    const float r_tx = 1.0f / (float)p.tiles_x;
    const int kxs = C::kTaps / KYS;
    const int n_kg = kxs / p.kxps;  // stages per channel chunk

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
                // per chunk q: one box {chunk, BN, taps} -> [tap][BN][chunk]
                mbar_expect_tx(bres, (uint32_t)(p.nq * C::kTaps) * p.b_tap);
                for (int q = 0; q < p.nq; ++q) {
                    const bool second = q >= p.nq0;
                    const int kc = second ? p.c0 + (q - p.nq0) * CHUNK : q * CHUNK;
                    tma_load_3d(smem + p.off_b + q * C::kTaps * p.b_tap, &mB, kc, 0, 0, bres);
                }
            }
            uint32_t it = 0;
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
                const ItemPos ip = item_pos(p, item, r_nt, r_tpi, r_tx, R);
                for (int q = 0; q < p.nq; ++q) {
                    const bool second = q >= p.nq0;
                    const int c = (second ? q - p.nq0 : q) * CHUNK;
                    const CUtensorMap *ma = second ? &mA1 : &mA0;
                    for (int kg = 0; kg < n_kg; ++kg, ++it) {
                        const int s = (int)(it % (uint32_t)S);
                        const uint32_t ph = (it / (uint32_t)S) & 1u;
                        mbar_wait(empty + s, ph ^ 1u);
                        uint8_t *st = smem + (size_t)s * p.stage_bytes;
                        const uint32_t btx = p.resident ? 0u : (uint32_t)(p.kxps * KYS) * p.b_tap;
                        mbar_expect_tx(full + s, p.a_tx + btx);
                        tma_load_4d(st, ma, c, ip.x0 - (C::kConv3 ? 1 : 0),
                                    ip.y0 - (C::kConv3 ? 1 : 0), ip.img, full + s);
                        if (!p.resident)
                            tma_load_3d(st + p.a_bytes, &mB, (second ? p.c0 : 0) + c, ip.nt * BN,
                                        kg * p.kxps * KYS, full + s);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------- MMA issuer -------------------------------
            const uint32_t idesc = idesc_bf16(128, BN);
            const uint64_t dproto = smem_desc(0, C::kRow, C::kLayout);
            const uint32_t dhi = (uint32_t)(dproto >> 32), dlo = (uint32_t)dproto;
            if (p.resident) mbar_wait(bres, 0);
            const uint32_t b_tap16 = p.b_tap >> 4;
            uint32_t it = 0, acc = 0;
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, ++acc) {
                const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
                mbar_wait(tempty + ab, aph ^ 1u);
                fence_after_sync();
                const uint32_t d0 = tmem + ab * C::kItemCols;
                for (int q = 0; q < p.nq; ++q) {
                    for (int kg = 0; kg < n_kg; ++kg, ++it) {
                        const int s = (int)(it % (uint32_t)S);
                        const uint32_t ph = (it / (uint32_t)S) & 1u;
                        mbar_wait(full + s, ph);
                        fence_after_sync();
                        const uint32_t st = sbase + (uint32_t)s * p.stage_bytes;
                        const uint32_t a_lo = dlo + (st >> 4);
                        // B row block of (kx, ky): resident [q][tap][BN], streamed [tap_in_stage][BN]
                        const uint32_t b_lo =
                            dlo + ((p.resident ? sbase + p.off_b + (uint32_t)(q * C::kTaps) * p.b_tap +
                                                     (uint32_t)(kg * p.kxps * KYS) * p.b_tap
                                               : st + p.a_bytes) >>
                                   4);
                        for (int k = 0; k < p.kxps; ++k) {
                            const int kx = kg * p.kxps + k;
#pragma unroll
                            for (int u = 0; u < MT; ++u) {
#pragma unroll
                                for (int ky = 0; ky < KYS; ++ky) {
#pragma unroll
                                    for (int j = 0; j < CHUNK / 16; ++j) {
                                        const uint32_t ao =
                                            ((u * 128 + ky * P + kx) * C::kRow + 32 * j) / 16;
                                        const uint32_t bo =
                                            (uint32_t)(k * KYS + ky) * b_tap16 + (32 * j) / 16;
                                        mma_bf16(d0 + u * BN, ((uint64_t)dhi << 32) | (a_lo + ao),
                                                 ((uint64_t)dhi << 32) | (b_lo + bo), idesc,
                                                 (q | kg | k | ky | j) != 0 ? 1u : 0u);
                                    }
                                }
                            }
                        }
                        mma_commit(empty + s);
                    }
                }
                mma_commit(tfull + ab);
            }
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        // GEMM row r = u*128 + m of an item is output pixel (r / P, r % P);
        // columns >= 16 and rows >= R are junk and discarded.
        const int eg = (warp - 2) >> 2;          // warpgroup -> every kEpiGroups-th item
        const int quarter = warp & 3;            // TMEM lane quarter this warp may access
        const int m = quarter * 32 + lane;
        const int et = threadIdx.x - 64 - 128 * eg;  // 0..127 within the warpgroup
        const uint32_t sstage = sbase + p.off_stage + (uint32_t)eg * p.stage_grp;
        uint32_t acc = (uint32_t)eg;
        for (int item = blockIdx.x + eg * gridDim.x; item < p.n_items;
             item += C::kEpiGroups * gridDim.x, acc += C::kEpiGroups) {
            const ItemPos ip = item_pos(p, item, r_nt, r_tpi, r_tx, R);
            const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
            mbar_wait(tfull + ab, aph);
            fence_after_sync();
            const uint32_t tbase = tmem + ab * C::kItemCols + ((uint32_t)(quarter * 32) << 16);
            float hacc[MT][4];
#pragma unroll
            for (int u = 0; u < MT; ++u)
#pragma unroll
                for (int j2 = 0; j2 < 4; ++j2) hacc[u][j2] = 0.0f;
#pragma unroll 1
            for (int g = 0; g < BN / 32; ++g) {
                const int n0 = ip.nt * BN + g * 32;
                if (n0 >= p.n_total) break;  // uniform
#pragma unroll 1
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int n = n0 + h2 * 16;
                    if (n >= p.n_total) break;  // uniform (n_total may be 16 mod 32)
#pragma unroll
                    for (int u = 0; u < MT; ++u) {
                        const int r = u * 128 + m;
                        const int yy = r / P, xx = r - yy * P;
                        const int gy = ip.y0 + yy, gx = ip.x0 + xx;
                        const bool valid = xx < kTW && yy < R && gx < p.w && gy < p.h;
                        uint32_t rr[16];
                        tmem_ld16(tbase + (uint32_t)(u * BN + g * 32 + h2 * 16), rr);
                        if (u + 1 == MT && (h2 == 1 || n + 16 >= p.n_total) &&
                            (g + 1 == BN / 32 || n0 + 32 >= p.n_total)) {
                            // item fully read -> hand the TMEM buffer back early
                            fence_before_sync();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(tempty + ab);
                        }
                        float v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            v[i] = apply_act(fmaf(__uint_as_float(rr[i]), s_scale[n + i],
                                                  s_shift[n + i]),
                                             p.act, p.alpha);
                        if (MODE == kHead) {
                            for (int j2 = 0; j2 < p.head_c; ++j2) {
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    hacc[u][j2] = fmaf(s_hw[j2 * p.cout + n + i], v[i], hacc[u][j2]);
                            }
                            if (!p.y && !p.y_f32) continue;  // head input not materialised
                        }
                        uint32_t pk[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                        if (valid) {
                            int64_t pix;
                            int o = n;
                            if (MODE == kTransposed) {
                                const int dd = n / p.cout;
                                o = n - dd * p.cout;
                                pix = ((int64_t)ip.img * (2 * p.h) + 2 * gy + (dd >> 1)) * (2 * p.w) +
                                      2 * gx + (dd & 1);
                            } else {
                                pix = ((int64_t)ip.img * p.h + gy) * p.w + gx;
                            }
                            if (p.y) {
                                uint4 *dst = reinterpret_cast<uint4 *>(p.y + pix * p.cout + o);
                                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
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
                            // stage this 16-channel slice of every GEMM row of the item
                            st_shared_v4(sstage + (uint32_t)r * 32u, make_uint4(pk[0], pk[1], pk[2], pk[3]));
                            st_shared_v4(sstage + (uint32_t)r * 32u + 16u,
                                         make_uint4(pk[4], pk[5], pk[6], pk[7]));
                        }
                    }
                    if (MODE == kPool) {
                        named_bar_sync(1 + eg, 128);
                        // (R/2) x 8 pooled outputs per item
                        for (int o = et; o < (R / 2) * (kTW / 2); o += 128) {
                            const int py = o >> 3, px = o & 7;
                            const int r00 = (2 * py) * P + 2 * px;
                            const int gy = ip.y0 + 2 * py, gx = ip.x0 + 2 * px;
                            if (gx >= p.w || gy >= p.h) continue;
                            uint4 o2[2];
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                const uint4 a0 = ld_shared_v4(sstage + (uint32_t)r00 * 32u + hh * 16);
                                const uint4 a1 = ld_shared_v4(sstage + (uint32_t)(r00 + 1) * 32u + hh * 16);
                                const uint4 a2 = ld_shared_v4(sstage + (uint32_t)(r00 + P) * 32u + hh * 16);
                                const uint4 a3 = ld_shared_v4(sstage + (uint32_t)(r00 + P + 1) * 32u + hh * 16);
                                o2[hh] = make_uint4(hmax4(a0.x, a1.x, a2.x, a3.x),
                                                    hmax4(a0.y, a1.y, a2.y, a3.y),
                                                    hmax4(a0.z, a1.z, a2.z, a3.z),
                                                    hmax4(a0.w, a1.w, a2.w, a3.w));
                            }
                            const int64_t pp =
                                ((int64_t)ip.img * (p.h / 2) + gy / 2) * (p.w / 2) + gx / 2;
                            uint4 *dst = reinterpret_cast<uint4 *>(p.pool + pp * p.cout + n);
                            dst[0] = o2[0];
                            dst[1] = o2[1];
                        }
                        named_bar_sync(1 + eg, 128);
                    }
                }
            }
            if (MODE == kHead) {
#pragma unroll
                for (int u = 0; u < MT; ++u) {
                    const int r = u * 128 + m;
                    const int yy = r / P, xx = r - yy * P;
                    const int gy = ip.y0 + yy, gx = ip.x0 + xx;
                    if (!(xx < kTW && yy < R && gx < p.w && gy < p.h)) continue;
                    const int64_t pix = ((int64_t)ip.img * p.h + gy) * p.w + gx;
                    for (int j2 = 0; j2 < p.head_c; ++j2) {
                        const float z = hacc[u][j2] + __ldg(p.head_b + j2);
                        p.head_out[pix * p.head_c + j2] = 1.0f / (1.0f + expf(-z));
                    }
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

// activations NHWC bf16, box {chunk, box_w columns, box_h rows, 1}
static bool encode_act(CUtensorMap *map, const void *base, int c, int w, int h, int batch,
                       int chunk, int box_w, int box_h) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
    cuuint32_t box[4] = {(cuuint32_t)chunk, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// weights [taps][n_total][ctot], box {chunk, bn, taps_per_box}
static bool encode_wts(CUtensorMap *map, const void *base, int ctot, int n_total, int taps,
                       int chunk, int bn, int taps_box) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)ctot, (cuuint64_t)n_total, (cuuint64_t)taps};
    cuuint64_t strides[2] = {(cuuint64_t)ctot * 2, (cuuint64_t)n_total * ctot * 2};
    cuuint32_t box[3] = {(cuuint32_t)chunk, (cuuint32_t)bn, (cuuint32_t)taps_box};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(chunk * 2),
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

namespace ls {
namespace unet {

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
    k_conv_p<BN, CHUNK, MODE><<<pl->grid, CfgP<BN, CHUNK, MODE>::kThreads, pl->smem, st>>>(
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

static int mt_for(int bn) { return bn <= 32 ? 4 : (bn <= 64 ? 2 : 1); }
static int rows_for(int bn, bool conv3, bool pool) {
    const int mt = mt_for(bn);
    if (!conv3) return 8 * mt;
    return (pool && (7 * mt) % 2) ? 7 * mt - 1 : 7 * mt;
}
static int epi_groups_for(int bn) {
    const int item_cols = mt_for(bn) * bn;
    const int acc = 512 / item_cols >= 4 ? 4 : 512 / item_cols;
    return acc >= 4 ? 3 : (acc >= 3 ? 2 : 1);
}

}  // namespace unet
}  // namespace ls

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
    if (!d_x0 || !d_w || !d_scale || !d_shift || batch < 1 || h < 1 || w < 1 || !chunk_ok(c0))
        return fail(LS_EINVAL);
    if (c1 < 0 || (c1 > 0 && (!d_x1 || !chunk_ok(c1)))) return fail(LS_EINVAL);
    if (cout < 16 || cout % 16 || (ksize != 1 && ksize != 3)) return fail(LS_EINVAL);
    if (transposed && (ksize != 1 || c1 != 0 || d_pool || d_head_w)) return fail(LS_EINVAL);
    if (!transposed && ksize != 3) return fail(LS_EINVAL);  // 1x1 convs are fused heads
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
    p.c0 = c0;
    p.c1 = c1;
    p.ctot = c0 + c1;
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
    const bool conv3 = !transposed;
    const int taps = conv3 ? 9 : 1, kys = conv3 ? 3 : 1, kxs = conv3 ? 3 : 1;
    const int pitch = conv3 ? 18 : 16;
    const size_t const_bytes = ((size_t)(2 * n_total + (d_head_w ? head_c * cout : 0)) * 4 + 1023) &
                               ~size_t(1023);
    size_t res_bytes = 0, stage_alloc = 0;
    int stages = 0;
    // Fit >= 3 pipeline stages: first all taps per stage, then one kx per
    // stage, then a narrower K chunk, then a narrower column tile.
    for (;;) {
        const int mt = mt_for(bn);
        const int rows = rows_for(bn, conv3, d_pool != nullptr);
        const int box_h = conv3 ? rows + 2 : rows;
        const uint32_t row = (uint32_t)chunk * 2;
        p.tiles_x = (w + kTW - 1) / kTW;
        p.tiles_y = (h + rows - 1) / rows;
        p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
        p.n_tiles_n = (n_total + bn - 1) / bn;
        p.n_items = p.n_tiles_m * p.n_tiles_n;
        p.nq0 = c0 / chunk;
        p.nq = (c0 + c1) / chunk;
        p.a_tx = (uint32_t)(pitch * box_h) * row;
        p.a_bytes = (p.a_tx + 1023u) & ~1023u;
        p.b_tap = (uint32_t)bn * row;
        p.resident = (p.n_tiles_n == 1 && (size_t)p.nq * taps * p.b_tap <= kResidentMax) ? 1 : 0;
        res_bytes = p.resident ? (size_t)p.nq * taps * p.b_tap : 0;
        stage_alloc = d_pool ? (size_t)epi_groups_for(bn) * (size_t)(mt * 128) * 32 : 0;
        const size_t fixed = res_bytes + const_bytes + stage_alloc + 512;
        bool fit = false;
        for (int kxps = kxs; kxps >= 1 && !fit; kxps = kxps == 1 ? 0 : 1) {
            const size_t raw = p.a_bytes + (p.resident ? 0 : (size_t)(kxps * kys) * p.b_tap);
            const size_t stage_bytes = (raw + 1023) & ~size_t(1023);
            stages = kSmemBudget > fixed ? (int)((kSmemBudget - fixed) / stage_bytes) : 0;
            if (stages >= 3) {
                p.kxps = kxps;
                p.stage_bytes = (uint32_t)stage_bytes;
                fit = true;
            }
        }
        if (fit) break;
        if (chunk > 16 && (c0 % (chunk / 2)) == 0 && (c1 % (chunk / 2)) == 0) {
            chunk >>= 1;
        } else if (bn > 32 && !d_head_w) {
            bn >>= 1;
        } else {
            delete pl;
            return fail(LS_EINVAL);
        }
    }
    if (stages > 8) stages = 8;
    p.stages = stages;
    p.off_b = (uint32_t)(stages * p.stage_bytes);
    p.off_const = (uint32_t)(p.off_b + res_bytes);
    p.off_stage = (uint32_t)(p.off_const + const_bytes);
    p.stage_grp = d_pool ? (uint32_t)(mt_for(bn) * 128 * 32) : 0;
    p.off_bar = (uint32_t)(p.off_stage + stage_alloc);
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = bn;
    pl->chunk = chunk;
    pl->mode = transposed ? kTransposed : (d_head_w ? kHead : (d_pool ? kPool : kPlain));
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    const int box_h = rows_for(bn, conv3, d_pool != nullptr) + (conv3 ? 2 : 0);
    bool ok = encode_act(&pl->a0, d_x0, c0, w, h, batch, chunk, pitch, box_h);
    ok = ok && encode_act(&pl->a1, c1 > 0 ? d_x1 : d_x0, c1 > 0 ? c1 : c0, w, h, batch, chunk,
                          pitch, box_h);
    ok = ok && encode_wts(&pl->b, d_w, p.ctot, n_total, taps, chunk, bn,
                          p.resident ? taps : p.kxps * kys);
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
