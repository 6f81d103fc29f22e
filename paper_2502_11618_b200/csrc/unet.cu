// U-Net convolutions on sm_100a tensor cores: implicit GEMM with TMA-fed
// operands, tcgen05.mma (kind::f16, bf16 x bf16 -> f32) with the accumulators
// in TMEM, and a fused epilogue (folded BatchNorm scale/shift, ReLU / leaky,
// 2x2 max pool, the final 1x1 conv + sigmoid, pixel-shuffle store of the 2x2
// transposed conv).
//
// GEMM view of one layer:  D[M = pixels][N = out channels] = A[M][K] * B[N][K]^T
//   A : im2col of the NHWC bf16 input, never materialised: TMA boxes of the
//       input whose out-of-bounds zero fill is the conv's "same" padding; the
//       decoder's [up, skip] concat is two tensor maps walked in K order.
//   B : the weights, K-major, layout [tap][n][c] with tap = kx*3 + ky.
//
// Kernel structure (persistent, warp-specialised, one CTA per SM):
//   warp 0 lane 0 : TMA producer over a STAGES-deep shared-memory ring
//   warp 1 lane 0 : tcgen05.mma issuer (descriptors precomputed: per MMA only
//                   the 14-bit start-address field moves, by constant offsets)
//   warps 2..     : kEpiGroups epilogue warpgroups; each drains a different
//                   work item (4 warps = the 4 TMEM lane quarters)
// A work item is MT x 128 output pixels (MT sub-tiles of 8 rows x 16 columns
// stacked vertically) times BN output columns; TMEM holds kAcc items' worth of
// accumulators so the MMA warp runs ahead of the epilogues.
// Halo reuse: for each channel chunk one TMA box of (8*MT + 2) rows x 16
// columns per kx serves all three ky taps and all MT sub-tiles -- tap ky /
// sub-tile u is the same smem box offset by (u*8 + ky)*16 rows, i.e. whole
// 8-row swizzle atoms, so only the descriptor start moves.
// Small weight tensors (<= kResidentMax, one column tile) stay resident in
// shared memory for the whole CTA; otherwise weight boxes stream with A.
#include <atomic>
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

// sub-tiles per work item of the 128 / 256-column tiles (A/B build switches)
// timing experiments only (scripts/exp builds; wrong outputs): pixel-pair stores
// almost never issued (the math stays live), C8 MMAs per item (0..3 ky rows)
#ifndef LS_EXP_PX_STORE_GUARD
#define LS_EXP_PX_STORE_GUARD
#endif
#ifndef LS_EXP_PX_C8_KY
#define LS_EXP_PX_C8_KY 3
#endif
#ifdef LS_EXP_NO_GDC
#define LS_GDC_WAIT() ((void)0)  // timing-only experiment: layers overlap unsafely
#else
#define LS_GDC_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#endif
#ifndef LS_MT128
#define LS_MT128 1
#endif
#ifndef LS_MT256
#define LS_MT256 1
#endif
// epilogue warpgroups that split ONE item's columns when an item fills TMEM
// (256-column tiles of two sub-tiles: the single-wave deep layers)
#ifndef LS_SPLIT_GROUPS
#define LS_SPLIT_GROUPS 3
#endif
// k_conv_px2 KX2 epilogue warpgroups (A/B build switch)
#ifndef LS_KX2_GROUPS
#define LS_KX2_GROUPS 3
#endif
// k_conv_px2 epilogue warpgroups of the 8-channel neighbour-row layer, e0c1 (A/B build switch)
#ifndef LS_C8_GROUPS
#define LS_C8_GROUPS 3
#endif
// k_conv_px2 KX2 epilogue warpgroups with 64 output channels (A/B build switch)
#ifndef LS_KX2_64_GROUPS
#define LS_KX2_64_GROUPS 2
#endif
// k_conv_kx (cout = 32): issue the second 16-channel half's TMEM loads before
// processing the first (A/B build switch)
#ifndef LS_KX_PIPE
#define LS_KX_PIPE 0
#endif

constexpr int kTW = 16, kTH = 8;
constexpr size_t kResidentMax = 80 * 1024;
// dynamic shared memory a plan may lay out (+ 1 KB alignment slack; the
// opt-in maximum is 227 KB) -- A/B build switch
#ifndef LS_SMEM_BUDGET_KB
#define LS_SMEM_BUDGET_KB 222
#endif
constexpr size_t kSmemBudget = LS_SMEM_BUDGET_KB * 1024;

enum EpiMode { kPlain = 0, kPool = 1, kHead = 2, kTransposed = 3 };

struct ConvParamsP {
    int batch, h, w;
    int tiles_x, tiles_y, n_tiles_m, n_tiles_n, n_items;
    int ty0;                // first tile row of a row band (ls_conv_plan_set_rows)
    int reverse;            // walk the tiles bottom-right first (ls_conv_plan_set_reverse)
    int pair_h;             // CTA pairs side by side (16-column offset) instead of stacked
    int c0, c1, ctot, nq0, nq;
    int kxs, kxps, pad;     // kx taps, kx taps per pipeline stage (1 or kxs)
    int n_total, cout, act;
    float alpha;
    const float *scale, *shift;
    __nv_bfloat16 *y;
    float *y_f32;
    __nv_bfloat16 *pool;
    const float *head_w, *head_b;
    int head_c;
    float *head_out;
    const void *wts;        // weights [tap][n][c] (k_conv_px2 C8 builds its B tiles from it)
    // k_conv_px2: the 32 columns' BN scale / shift as kernel parameters (copied at
    // plan creation) -- the epilogue reads them as constant-bank operands instead
    // of shared-memory loads, which competed with the MMA operand reads in L1
    float pc_scale[64], pc_shift[64];
    float pc_head[4 * 32];  // k_conv_px2 head: the final 1x1 conv's weights [head_c][32]
    float pc_upb[32];       // k_conv_upfuse: the fused transposed conv's bias
    int resident;           // weights resident in smem
    int stages;
    uint32_t a_bytes;       // one A box footprint (1024-aligned)
    uint32_t a_tx;          // TMA bytes of one A box
    uint32_t b_blk;         // bytes of one (3 x BN x chunk) weight block
    uint32_t stage_bytes;
    uint32_t off_b;         // resident weights
    uint32_t off_const;     // scale[n_total], shift[n_total], head_w (f32)
    uint32_t off_pool;      // (unused: pooling is done with warp shuffles)
    uint32_t off_bar;       // barriers
    // transposed convs with 32 output channels: each epilogue group stages its
    // item's 16x32-pixel output tile (32 KB, 128 B swizzle) at off_stage + 32 KB*eg
    // and writes it with one TMA store (pixel-shuffle lanes otherwise store 32 B
    // chunks 128 B apart, ~32 L1 wavefronts per store instruction)
    int stage_store;
    uint32_t off_stage;
};

// 128-pixel sub-tiles per work item: more sub-tiles share each streamed
// weight stage (a 256-column layer reads 48 KB of weights per 10 KB of
// activations), fewer items fill the 148 SMs -- the plan picks 2 for
// 256-column tiles when that still leaves >= ~0.8 items per SM
constexpr int default_mt(int bn) {
    return bn <= 32 ? 4 : (bn <= 64 ? 2 : (bn <= 128 ? LS_MT128 : LS_MT256));
}

template <int BN, int CHUNK, int MT = default_mt(BN)>
struct CfgP {
    static constexpr uint32_t kRow = CHUNK * 2;  // bytes per operand row
    static constexpr uint32_t kLayout =
        CHUNK == 64 ? kSwizzle128B : (CHUNK == 32 ? kSwizzle64B : kSwizzle32B);
    static constexpr int kMT = MT;
    static constexpr int kItemCols = kMT * BN;                          // TMEM columns per item
    static constexpr int kAcc = 512 / kItemCols >= 4 ? 4 : 512 / kItemCols;
    // kAcc == 1: the MMA warp cannot run ahead of the epilogue, so several
    // warpgroups drain the SAME item, each a share of its 32-column groups
    static constexpr bool kSplit = kAcc == 1 && LS_SPLIT_GROUPS > 1;
    static constexpr int kEpiGroups =
        kSplit ? LS_SPLIT_GROUPS : (kAcc >= 4 ? 3 : (kAcc >= 3 ? 2 : 1));
    static constexpr int kThreads = 64 + 128 * kEpiGroups;
    static constexpr int kTmemCols = kAcc * kItemCols <= 32 ? 32 :
                                     (kAcc * kItemCols <= 64 ? 64 :
                                     (kAcc * kItemCols <= 128 ? 128 :
                                     (kAcc * kItemCols <= 256 ? 256 : 512)));
    static constexpr int kGroups = BN / 16;
};

template <int BN, int CHUNK, int MT>
constexpr int threads_for() { return CfgP<BN, CHUNK, MT>::kThreads; }

// Branch-free activation: max(v, slope * v) with slope 0 (ReLU), alpha (leaky,
// 0 <= alpha <= 1) or 1 (none) -- the layer's slope is resolved once.
__device__ __forceinline__ float act_slope(int act, float alpha) {
    return act == LS_ACT_RELU ? 0.0f : (act == LS_ACT_LEAKY ? alpha : 1.0f);
}

__device__ __forceinline__ float apply_act(float v, float slope) { return fmaxf(v, slope * v); }

// Packed f32x2 arithmetic (FADD2 / FFMA2 / FMUL2 on sm_100): two channels per
// instruction with exactly the scalar ops' IEEE results, so the packed
// epilogue computes bit-identical values with fewer issue slots.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unf2(f32x2 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// apply_act on a channel pair: max(v, slope * v)
__device__ __forceinline__ void act2(f32x2 y, f32x2 slope2, float &a, float &b) {
    float c, d;
    unf2(y, a, b);
    unf2(mul2(y, slope2), c, d);
    a = fmaxf(a, c);
    b = fmaxf(b, d);
}

// Output sigmoid (FE:model/grad64.ts:343) with the fast exp / divide: a few
// ulp of f32 -- far inside the bf16 network's tolerance -- for ~1/3 of the
// instructions of expf + an IEEE division (which were a quarter of the head
// layer's issue slots).  exp overflow gives 1/inf = 0, underflow 1/1 = 1.
__device__ __forceinline__ float sigmoid_fast(float z) {
    return __fdividef(1.0f, 1.0f + __expf(-z));
}

__device__ __forceinline__ uint32_t hmax2u(uint32_t a, uint32_t b) {
    __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162 *>(&a);
    __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162 *>(&b);
    __nv_bfloat162 m = __hmax2(x, y);
    return *reinterpret_cast<uint32_t *>(&m);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

// Final 1x1 conv partial sums over 16 channels (same sequential FMA order
// per output as a scalar loop; weights read as float4 broadcasts).
__device__ __forceinline__ void head_accumulate(const float *s_hw, int cout, int head_c, int n,
                                                const float (&v)[16], float (&hacc)[4]) {
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
        if (j2 >= head_c) break;
        const float4 *w4 = reinterpret_cast<const float4 *>(s_hw + j2 * cout + n);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 w = w4[q];
            hacc[j2] = fmaf(w.x, v[4 * q], hacc[j2]);
            hacc[j2] = fmaf(w.y, v[4 * q + 1], hacc[j2]);
            hacc[j2] = fmaf(w.z, v[4 * q + 2], hacc[j2]);
            hacc[j2] = fmaf(w.w, v[4 * q + 3], hacc[j2]);
        }
    }
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

// Work-item position as a mixed-radix counter (n-tile, tile x, tile y,
// image), advanced by a fixed stride without divisions: a persistent CTA walks
// items blockIdx.x, +gridDim.x, ... and each step's position came from three
// f32-reciprocal divisions (conversion latency on every item).
struct ItemWalk {
    int nt, tx, ty, img;
    int s_nt, s_tx, s_ty, s_img;
    __device__ static void digits(const ConvParamsP &p, int v, int &a, int &b, int &c, int &d) {
        a = v % p.n_tiles_n;
        v /= p.n_tiles_n;
        b = v % p.tiles_x;
        v /= p.tiles_x;
        c = v % p.tiles_y;
        d = v / p.tiles_y;
    }
    __device__ void init(const ConvParamsP &p, int item, int stride) {
        digits(p, item, nt, tx, ty, img);
        digits(p, stride, s_nt, s_tx, s_ty, s_img);
    }
    __device__ void next(const ConvParamsP &p) {
        nt += s_nt;
        int c = nt >= p.n_tiles_n;
        nt -= c * p.n_tiles_n;
        tx += s_tx + c;
        c = tx >= p.tiles_x;
        tx -= c * p.tiles_x;
        ty += s_ty + c;
        c = ty >= p.tiles_y;
        ty -= c * p.tiles_y;
        img += s_img + c;
    }
    // tile coordinates in traversal order: reversed plans visit the last tile
    // first, so a layer consumes its producer's most recently written (still
    // L2-resident) rows first when consecutive layers alternate direction
    __device__ int TX(const ConvParamsP &p) const { return p.reverse ? p.tiles_x - 1 - tx : tx; }
    __device__ int TY(const ConvParamsP &p) const { return p.reverse ? p.tiles_y - 1 - ty : ty; }
    __device__ int IMG(const ConvParamsP &p) const { return p.reverse ? p.batch - 1 - img : img; }
    __device__ ItemPos pos(const ConvParamsP &p, int tile_h, int tile_w = kTW) const {
        ItemPos ip;
        ip.nt = nt;
        ip.img = IMG(p);
        ip.y0 = (p.ty0 + TY(p)) * tile_h;
        ip.x0 = TX(p) * tile_w;
        return ip;
    }
};

// PAIR: a cluster of two CTAs on one TPC shares each M = 256 MMA (tcgen05
// cta_group::2, issued by the leader): CTA r holds the A rows of sub-tile
// rows [r*8*MT, (r+1)*8*MT) of a (16*MT)-row tile and output columns
// [r*BN/2, (r+1)*BN/2) of the B tile, and drains its own 128 TMEM lanes x BN
// columns.  Per SM the tensor core then reads 128 x 16 A + (BN/2) x 16 B per
// MMA instead of 128 x 16 + BN x 16: the 1-SM 128-column layers were bound
// by that shared-memory read traffic (A 4 KB + B 4 KB per 64-cycle MMA plus
// the TMA fills on a 128 B/cycle SRAM).
template <int BN, int CHUNK, int MODE, int MT_ = default_mt(BN), bool PAIR = false>
__global__ void __launch_bounds__(threads_for<BN, CHUNK, MT_>()) k_conv_p(
    const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
    const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mY,
    const ConvParamsP p) {
    using C = CfgP<BN, CHUNK, MT_>;
    if constexpr ((C::kSplit && !(MODE == kPlain || MODE == kPool)) ||
                  (PAIR && (C::kSplit || !(MODE == kPlain || MODE == kPool)))) {
        __trap();  // never planned: transposed tiles cap at 128 columns, heads use k_conv_px2
    } else {
    constexpr int KYS = MODE == kTransposed ? 1 : 3;
    constexpr int MT = C::kMT;
    // rows / columns per work item (both CTAs of a pair: stacked rows, or side by
    // side columns when p.pair_h)
    const int kTileH = kTH * MT * (PAIR && !p.pair_h ? 2 : 1);
    const int kTileW = kTW * (PAIR && p.pair_h ? 2 : 1);
    constexpr int kBNL = PAIR ? BN / 2 : BN;            // B columns held by this CTA
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    // work index / stride: pairs walk the items as one unit
    const int wid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int wstride = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
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
    const int n_kg = p.kxs / p.kxps;  // stages per channel chunk

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Programmatic dependent launch: let the next layer's CTAs start their own
    // prologue as SMs free up; everything this kernel does before
    // griddepcontrol.wait (barriers, TMEM, weights, epilogue constants) reads
    // only data no earlier kernel writes.
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, 1);
            }
            for (int a = 0; a < C::kAcc; ++a) {
                mbar_init(tfull + a, 1);
                mbar_init(tempty + a, 4 * (C::kSplit ? C::kEpiGroups : 1) * (PAIR ? 2 : 1));
            }
            mbar_init(bres, 1);
            fence_barrier_init();
            tma_prefetch(&mA0);
            if (p.c1 > 0) tma_prefetch(&mA1);
            tma_prefetch(&mB);
        }
        __syncwarp();
        if constexpr (PAIR)
            tmem_alloc_pair(tslot, C::kTmemCols);
        else
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
    if constexpr (PAIR)
        cluster_sync_all();  // the peer signals the leader's barriers from here on
    else
        __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    // the leader's barriers as shared::cluster addresses (PAIR: both CTAs' TMA
    // bytes complete on the leader's full / bres barriers, both CTAs' epilogues
    // release the leader's tempty)
    const uint32_t c_full = PAIR ? mapa_shared(full, 0) : 0u;
    const uint32_t c_bres = PAIR ? mapa_shared(bres, 0) : 0u;
    const uint32_t c_tempty = PAIR ? mapa_shared(tempty, 0) : 0u;

    if (warp == 0) {
        if (elect_one()) {
            // ------------------------------ TMA producer ------------------------------
            if (p.resident) {
                if (leader)
                    mbar_expect_tx(bres, (uint32_t)(p.kxs * p.nq) * p.b_blk * (PAIR ? 2u : 1u));
                for (int q = 0; q < p.nq; ++q)
                    for (int kx = 0; kx < p.kxs; ++kx) {
                        const bool second = q >= p.nq0;
                        const int kc = second ? p.c0 + (q - p.nq0) * CHUNK : q * CHUNK;
                        if constexpr (PAIR)
                            tma_load_3d_pair(smem + p.off_b + (q * p.kxs + kx) * p.b_blk, &mB, kc,
                                             (int)rank * kBNL, kx * KYS, c_bres);
                        else
                            tma_load_3d(smem + p.off_b + (q * p.kxs + kx) * p.b_blk, &mB, kc, 0,
                                        kx * KYS, bres);
                    }
            }
            // the previous layer's activations are complete and visible past here;
            // every global write of this kernel depends on loads issued after it
            LS_GDC_WAIT();
            int s = 0;
            uint32_t ph = 0;
            ItemWalk walk;
            walk.init(p, wid, wstride);
            // this CTA's first row / column in the item
            const int ry = PAIR && !p.pair_h ? (int)rank * kTH * MT : 0;
            const int rx = PAIR && p.pair_h ? (int)rank * kTW : 0;
            for (int item = wid; item < p.n_items; item += wstride, walk.next(p)) {
                const ItemPos ip = walk.pos(p, kTileH, kTileW);
                for (int q = 0; q < p.nq; ++q) {
                    const bool second = q >= p.nq0;
                    const int c = (second ? q - p.nq0 : q) * CHUNK;
                    const CUtensorMap *ma = second ? &mA1 : &mA0;
                    for (int kg = 0; kg < n_kg; ++kg, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                        mbar_wait(empty + s, ph ^ 1u);
                        uint8_t *st = smem + (size_t)s * p.stage_bytes;
#ifdef LS_EXP_B_ONCE
                        // timing-only experiment: stream the weights for the first item only
                        const bool load_b = !p.resident && item == wid;
#else
                        const bool load_b = !p.resident;
#endif
                        if (leader)
                            mbar_expect_tx(full + s, p.kxps * (p.a_tx + (load_b ? p.b_blk : 0u)) *
                                                         (PAIR ? 2u : 1u));
                        for (int k = 0; k < p.kxps; ++k) {
                            const int kx = kg * p.kxps + k;
                            if constexpr (PAIR) {
                                const uint32_t cb = c_full + 8u * (uint32_t)s;
                                tma_load_4d_pair(st + k * p.a_bytes, ma, c, ip.x0 + rx + kx - p.pad,
                                                 ip.y0 + ry - p.pad, ip.img, cb);
                                if (load_b)
                                    tma_load_3d_pair(st + p.kxps * p.a_bytes + k * p.b_blk, &mB,
                                                     (second ? p.c0 : 0) + c,
                                                     ip.nt * BN + (int)rank * kBNL, kx * KYS, cb);
                            } else {
                                tma_load_4d(st + k * p.a_bytes, ma, c, ip.x0 + kx - p.pad,
                                            ip.y0 - p.pad, ip.img, full + s);
                                if (load_b)
                                    tma_load_3d(st + p.kxps * p.a_bytes + k * p.b_blk, &mB,
                                                (second ? p.c0 : 0) + c, ip.nt * BN, kx * KYS,
                                                full + s);
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && elect_one()) {
            // ------------------------------- MMA issuer -------------------------------
            const uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BN);
            const uint64_t dproto = smem_desc(0, C::kRow, C::kLayout);
            const uint32_t dhi = (uint32_t)(dproto >> 32), dlo = (uint32_t)dproto;
            if (p.resident) mbar_wait(bres, 0);
            const uint32_t a_box16 = p.a_bytes >> 4, b_blk16 = p.b_blk >> 4;
            int s = 0;
            uint32_t ph = 0, ab = 0, aph = 0;
            for (int item = wid; item < p.n_items;
                 item += wstride, ab = ab + 1 == C::kAcc ? 0 : ab + 1, aph ^= ab == 0) {
                mbar_wait(tempty + ab, aph ^ 1u);
                fence_after_sync();
                const uint32_t d0 = tmem + ab * C::kItemCols;
                for (int q = 0; q < p.nq; ++q) {
                    for (int kg = 0; kg < n_kg; ++kg, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                        mbar_wait(full + s, ph);
                        fence_after_sync();
                        const uint32_t st = sbase + (uint32_t)s * p.stage_bytes;
                        const uint32_t a_lo = dlo + (st >> 4);
                        const uint32_t b_lo =
                            dlo + ((p.resident
                                        ? sbase + p.off_b + (uint32_t)(q * p.kxs + kg * p.kxps) * p.b_blk
                                        : st + p.kxps * p.a_bytes) >>
                                   4);
                        // (scripts/mma_rate.cu: a 128xNx16 MMA costs max(~45, N/2)
                        // cycles whatever the accumulator order -- N=32 tiles top
                        // out at 36% of the tensor peak)
                        for (int k = 0; k < p.kxps; ++k) {
#pragma unroll
                            for (int u = 0; u < MT; ++u) {
#pragma unroll
                                for (int ky = 0; ky < KYS; ++ky) {
#pragma unroll
                                    for (int j = 0; j < CHUNK / 16; ++j) {
                                        const uint32_t ao =
                                            k * a_box16 + ((u * kTH + ky) * kTW * C::kRow + 32 * j) / 16;
                                        const uint32_t bo = k * b_blk16 + (ky * kBNL * C::kRow + 32 * j) / 16;
                                        const uint64_t ad = ((uint64_t)dhi << 32) | (a_lo + ao);
                                        const uint64_t bd = ((uint64_t)dhi << 32) | (b_lo + bo);
                                        const uint32_t acc = (q | kg | k | ky | j) != 0 ? 1u : 0u;
                                        if constexpr (PAIR)
                                            mma_bf16_pair(d0 + u * BN, ad, bd, idesc, acc);
                                        else
                                            mma_bf16(d0 + u * BN, ad, bd, idesc, acc);
                                    }
                                }
                            }
                        }
                        if constexpr (PAIR)
                            mma_commit_pair(empty + s);
                        else
                            mma_commit(empty + s);
                    }
                }
                if constexpr (PAIR)
                    mma_commit_pair(tfull + ab);
                else
                    mma_commit(tfull + ab);
            }
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        // Pixel m = quarter*32 + lane of a sub-tile is (row m/16, col m%16): the
        // 2x2 max-pool partners of a lane are lanes ^1 and ^16 of the SAME warp,
        // so pooling is two shuffle-max steps (no shared memory, no barriers).
        const int eg = (warp - 2) >> 2;          // warpgroup -> every kEpiGroups-th item
        const int quarter = warp & 3;            // TMEM lane quarter this warp may access
        const int m = quarter * 32 + lane;
        const int tx = m % kTW, ty = m / kTW;
        const float slope = act_slope(p.act, p.alpha);
        const f32x2 slope2 = f2(slope, slope);
        const float r_cout = 1.0f / (float)p.cout;
        // items per group: every kEpiGroups-th item, or (kSplit) every item
        constexpr int kItemGroups = C::kSplit ? 1 : C::kEpiGroups;
        const int eg_item = C::kSplit ? 0 : eg;
        uint32_t acc = (uint32_t)eg_item;
        ItemWalk walk;
        walk.init(p, wid + eg_item * wstride, kItemGroups * wstride);
        const int ry = PAIR && !p.pair_h ? (int)rank * kTH * MT : 0;  // this CTA's first
        const int rx = PAIR && p.pair_h ? (int)rank * kTW : 0;          // row / column
        for (int item = wid + eg_item * wstride; item < p.n_items;
             item += kItemGroups * wstride, acc += kItemGroups, walk.next(p)) {
            const ItemPos ip = walk.pos(p, kTileH, kTileW);
            const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
            mbar_wait(tfull + ab, aph);
            fence_after_sync();
            const uint32_t tbase = tmem + ab * C::kItemCols + ((uint32_t)(quarter * 32) << 16);
            const int gx = ip.x0 + rx + tx;
            // 32-column groups of this item that hold real columns (n_total may
            // end mid-tile, or be 16 mod 32)
            const int rem = p.n_total - ip.nt * BN;
            const int ng = rem >= BN ? BN / 32 : (rem + 31) / 32;
            const int steps = MT * ng;
            float hacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            // one 32-column group: scale/shift/act, bf16 pack, 32 B stores,
            // pooling / head as the mode asks
            auto process = [&](int u, int g, const uint32_t(&rr)[32]) {
                const int gy = ip.y0 + ry + u * kTH + ty;
                const bool valid = gx < p.w && gy < p.h;
                const int n0 = ip.nt * BN + g * 32;
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int n = n0 + h2 * 16;
                    if (n >= p.n_total) break;  // uniform (n_total may be 16 mod 32)
                    const float4 *sc4 = reinterpret_cast<const float4 *>(s_scale + n);
                    const float4 *sh4 = reinterpret_cast<const float4 *>(s_shift + n);
                    float v[16];
#pragma unroll
                    for (int i4 = 0; i4 < 4; ++i4) {
                        const float4 sc = sc4[i4], sh = sh4[i4];
                        const f32x2 sc2[2] = {f2(sc.x, sc.y), f2(sc.z, sc.w)};
                        const f32x2 sh2[2] = {f2(sh.x, sh.y), f2(sh.z, sh.w)};
#pragma unroll
                        for (int jp = 0; jp < 2; ++jp) {
                            const int i = 4 * i4 + 2 * jp;
                            const f32x2 x = f2(__uint_as_float(rr[h2 * 16 + i]),
                                               __uint_as_float(rr[h2 * 16 + i + 1]));
                            act2(fma2(x, sc2[jp], sh2[jp]), slope2, v[i], v[i + 1]);
                        }
                    }
                    if (MODE == kHead) {
                        head_accumulate(s_hw, p.cout, p.head_c, n, v, hacc);
                        if (!p.y && !p.y_f32) continue;  // head input not materialised
                    }
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                    if (MODE == kTransposed && p.stage_store) {
                        // cout 32: staging tile row (2*ty + dy)*16 + tx, 128 B per row
                        // holding [dx][32 channels]; cout 64 (the item covers one dy =
                        // its n-tile): row (ty*16 + tx)*2 + dx holding 64 channels.
                        // 16 B chunks XOR-swizzled by row (TMA 128 B)
                        int r, c;
                        if (p.cout == 64) {
                            r = (ty * kTW + tx) * 2 + ((n >> 6) & 1);
                            c = (n & 63) >> 3;
                        } else {
                            const int dd = n >> 5, dy = dd >> 1, dx = dd & 1;
                            r = (2 * ty + dy) * kTW + tx;
                            c = dx * 4 + ((n & 31) >> 3);
                        }
                        uint8_t *row = smem + p.off_stage + (uint32_t)eg * 32768u + r * 128;
                        *reinterpret_cast<uint4 *>(row + ((c ^ (r & 7)) << 4)) =
                            make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        *reinterpret_cast<uint4 *>(row + (((c + 1) ^ (r & 7)) << 4)) =
                            make_uint4(pk[4], pk[5], pk[6], pk[7]);
                        continue;
                    }
                    if (valid) {
                        int64_t pix;
                        int o = n;
                        if (MODE == kTransposed) {
                            // sub-pixel (dy, dx) of column n: one f32-reciprocal
                            // division (the integer one is ~20 dependent instructions)
                            const int dd = fdiv(n, p.cout, r_cout);
                            o = n - dd * p.cout;
                            pix = ((int64_t)ip.img * (2 * p.h) + 2 * gy + (dd >> 1)) * (2 * p.w) +
                                  2 * gx + (dd & 1);
                        } else {
                            pix = ((int64_t)ip.img * p.h + gy) * p.w + gx;
                        }
                        if (p.y) st_global_v8(p.y + pix * p.cout + o, pk);
                        if (p.y_f32) {
                            float4 *dst = reinterpret_cast<float4 *>(p.y_f32 + pix * p.cout + o);
                            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                            dst[2] = make_float4(v[8], v[9], v[10], v[11]);
                            dst[3] = make_float4(v[12], v[13], v[14], v[15]);
                        }
                    }
                    if (MODE == kPool) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            // horizontal pair (lane ^ 1), then vertical (lane ^ 16): two
                            // shuffles per word (max is exact and order-free)
                            const uint32_t a = hmax2u(pk[i], __shfl_xor_sync(0xffffffffu, pk[i], 1));
                            pk[i] = hmax2u(a, __shfl_xor_sync(0xffffffffu, a, 16));
                        }
                        if (valid && (lane & 17) == 0) {
                            const int64_t pp =
                                ((int64_t)ip.img * (p.h / 2) + gy / 2) * (p.w / 2) + gx / 2;
                            st_global_v8(p.pool + pp * p.cout + n, pk);
                        }
                    }
                }
                if (MODE == kHead && g + 1 == ng) {
                    if (valid) {
                        const int64_t pix = ((int64_t)ip.img * p.h + gy) * p.w + gx;
                        for (int j2 = 0; j2 < p.head_c; ++j2) {
                            const float z = hacc[j2] + __ldg(p.head_b + j2);
                            p.head_out[pix * p.head_c + j2] = sigmoid_fast(z);
                        }
                    }
                    hacc[0] = hacc[1] = hacc[2] = hacc[3] = 0.0f;
                }
            };
            // the TMEM buffer goes back to the MMA warp as soon as its last
            // group is in registers
            auto release = [&]() {
                fence_before_sync();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR)
                        mbar_arrive_cluster(c_tempty + 8u * ab);
                    else
                        mbar_arrive(tempty + ab);
                }
            };
            // two register buffers: group s+1's tcgen05.ld is in flight while
            // group s is processed
            uint32_t ra[32], rb[32];
            // (sub-tile, column group) of steps s and s+1, advanced without
            // integer division (ng is a runtime value)
            auto adv = [&](int &u, int &g) {
                if (++g == ng) {
                    g = 0;
                    ++u;
                }
            };
            auto colug = [&](int u, int g) -> uint32_t {
                return tbase + (uint32_t)(u * BN + g * 32);
            };
            if constexpr (C::kSplit && (MODE == kPlain || MODE == kPool)) {
                // (split epilogues keep per-column work only: no head sums, no
                // staged transposed stores -- those plans never use these tiles)
                // this group's steps: eg, eg + G, ... (step -> sub-tile, group)
                constexpr int G = C::kEpiGroups;
                auto ug = [&](int st, int &u, int &g) {
                    u = st / ng;
                    g = st - u * ng;
                };
                int st = eg, u = 0, g = 0;
                if (st >= steps) {
                    release();
                } else {
                    ug(st, u, g);
                    tmem_ld32_async(colug(u, g), ra);
                }
#pragma unroll 1
                while (st < steps) {
                    int un = 0, gn = 0;
                    const int sn = st + G;
                    tmem_ld_wait(ra);
                    if (sn < steps) {
                        ug(sn, un, gn);
                        tmem_ld32_async(colug(un, gn), rb);
                    } else {
                        release();
                    }
                    process(u, g, ra);
                    if (sn >= steps) break;
                    const int s2 = sn + G;
                    int u2 = 0, g2 = 0;
                    tmem_ld_wait(rb);
                    if (s2 < steps) {
                        ug(s2, u2, g2);
                        tmem_ld32_async(colug(u2, g2), ra);
                    } else {
                        release();
                    }
                    process(un, gn, rb);
                    st = s2;
                    u = u2;
                    g = g2;
                }
                continue;
            }
            int u0 = 0, g0 = 0, u1 = 0, g1 = 0;
            adv(u1, g1);
            tmem_ld32_async(colug(0, 0), ra);
#pragma unroll 1
            for (int s = 0; s < steps; s += 2) {
                int u2 = u1, g2 = g1;
                adv(u2, g2);  // step s + 2
                tmem_ld_wait(ra);
                if (s + 1 < steps) tmem_ld32_async(colug(u1, g1), rb);
                else release();
                process(u0, g0, ra);
                if (s + 1 < steps) {
                    tmem_ld_wait(rb);
                    if (s + 2 < steps) tmem_ld32_async(colug(u2, g2), ra);
                    else release();
                    process(u1, g1, rb);
                }
                u0 = u2;
                g0 = g2;
                u1 = u2;
                g1 = g2;
                adv(u1, g1);  // step s + 3
            }
            if (MODE == kTransposed && p.stage_store) {
                // the group's tile is complete: one TMA store, then the staging
                // buffer is reusable once the store has read it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                named_bar_sync(1 + eg, 128);
                if (quarter == 0 && lane == 0) {
                    if (p.cout == 64)  // [c][dx][j][dy][image * h_in + i], dy = n-tile
                        tma_store_5d(&mY, smem + p.off_stage + (uint32_t)eg * 32768u, 0, 0, ip.x0,
                                     ip.nt, ip.img * p.h + ip.y0);
                    else
                        tma_store_5d(&mY, smem + p.off_stage + (uint32_t)eg * 32768u, 0, ip.x0, 0,
                                     ip.y0, ip.img);
                    tma_store_wait_read();
                }
                named_bar_sync(1 + eg, 128);
            }
        }
    }
    if (MODE == kTransposed && p.stage_store && warp >= 2 && (warp & 3) == 0 && lane == 0)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
    fence_before_sync();
    if constexpr (PAIR) {
        // the leader's MMAs write the peer's TMEM and the peer's epilogue
        // arrives on the leader's barriers: neither CTA leaves before both are done
        cluster_sync_all();
        if (warp == 0) tmem_dealloc_pair(tmem, C::kTmemCols);
    } else {
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
    }
    }  // (planned modes)
}

// ---------------------------------------------------------------------------
// cout = 32 convolutions (the four full-resolution layers).  A 128xNx16 MMA
// costs max(~45, ~40 + N/4) cycles (scripts/mma_rate.cu), so N = 32 tiles run
// at 36% of the tensor peak at best.  Here the three kx taps are stacked
// along N ([kx][co], N = 96) -- each A operand read now feeds 96 columns --
// and the kx sum moves to the epilogue:
//     out(r, c) = T0(r, c-1) + T1(r, c) + T2(r, c+1)
// with lanes c +- 1 of the same 16-lane pixel row (warp shuffles).  A tile is
// 8 rows x 16 columns of INPUT pixels whose columns 1..14 are outputs (tiles
// advance by 14 columns); ky stays a descriptor row offset into one (8+2) x 16
// TMA box per K chunk.  Per K chunk: 3 MMAs of ~56 cycles instead of 9 of
// ~46, and one halo box instead of three.  Weights stay resident, loaded as
// nine 32-row blocks from the ABI's [tap][n][c] layout.
constexpr int kKxCols = 14;  // output columns per tile

template <int CHUNK, int COUT>
struct CfgKx {
    static constexpr uint32_t kRow = CHUNK * 2;
    static constexpr uint32_t kLayout =
        CHUNK == 64 ? kSwizzle128B : (CHUNK == 32 ? kSwizzle64B : kSwizzle32B);
    static constexpr int kN = 3 * COUT;                  // [kx][co]: 96 or 192 columns
    static constexpr int kAcc = 480 / kN;                // TMEM buffers: 5 or 2
    // (LS_KX_PIPE: 48 more live registers per thread -> at most 3 groups)
    static constexpr int kEpiGroups = (LS_KX_PIPE == 1 && COUT == 32) ? (kAcc >= 3 ? 3 : kAcc)
                                                                      : (kAcc >= 4 ? 4 : kAcc);
    static constexpr int kThreads = 64 + 128 * kEpiGroups;
    static constexpr int kTmemCols = 512;
};

template <int CHUNK, int COUT, int MODE>
__global__ void __launch_bounds__(CfgKx<CHUNK, COUT>::kThreads) k_conv_kx(
    const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
    const __grid_constant__ CUtensorMap mB, const ConvParamsP p) {
    using C = CfgKx<CHUNK, COUT>;
    extern __shared__ uint8_t smem_raw[];
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

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
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
        if (elect_one()) {
            // ------------------------------ TMA producer ------------------------------
            // resident weights: block (q, ky) = 3*COUT rows [kx][co], from taps kx*3+ky
            mbar_expect_tx(bres, (uint32_t)(9 * p.nq) * p.b_blk);
            for (int q = 0; q < p.nq; ++q) {
                const bool second = q >= p.nq0;
                const int kc = second ? p.c0 + (q - p.nq0) * CHUNK : q * CHUNK;
                for (int ky = 0; ky < 3; ++ky)
                    for (int kx = 0; kx < 3; ++kx)
                        tma_load_3d(smem + p.off_b + ((q * 3 + ky) * 3 + kx) * p.b_blk, &mB, kc, 0,
                                    kx * 3 + ky, bres);
            }
            LS_GDC_WAIT();
            int s = 0;
            uint32_t ph = 0;
            ItemWalk walk;
            walk.init(p, blockIdx.x, gridDim.x);
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, walk.next(p)) {
                const int img = walk.IMG(p), x0 = walk.TX(p) * kKxCols, y0 = (p.ty0 + walk.TY(p)) * kTH;
                for (int q = 0; q < p.nq; ++q, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                    const bool second = q >= p.nq0;
                    const int c = (second ? q - p.nq0 : q) * CHUNK;
                    mbar_wait(empty + s, ph ^ 1u);
                    mbar_expect_tx(full + s, p.a_tx);
                    tma_load_4d(smem + (size_t)s * p.stage_bytes, second ? &mA1 : &mA0, c, x0 - 1,
                                y0 - 1, img, full + s);
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            // ------------------------------- MMA issuer -------------------------------
            const uint32_t idesc = idesc_bf16(128, C::kN);
            const uint64_t dproto = smem_desc(0, C::kRow, C::kLayout);
            const uint32_t dhi = (uint32_t)(dproto >> 32), dlo = (uint32_t)dproto;
            mbar_wait(bres, 0);
            int s = 0;
            uint32_t ph = 0, ab = 0, aph = 0;
            for (int item = blockIdx.x; item < p.n_items;
                 item += gridDim.x, ab = ab + 1 == C::kAcc ? 0 : ab + 1, aph ^= ab == 0) {
                mbar_wait(tempty + ab, aph ^ 1u);
                fence_after_sync();
                const uint32_t d0 = tmem + ab * C::kN;
                for (int q = 0; q < p.nq; ++q, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                    mbar_wait(full + s, ph);
                    fence_after_sync();
                    const uint32_t a_lo = dlo + ((sbase + (uint32_t)s * p.stage_bytes) >> 4);
                    const uint32_t b_lo = dlo + ((sbase + p.off_b + (uint32_t)(q * 9) * p.b_blk) >> 4);
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
#pragma unroll
                        for (int j = 0; j < CHUNK / 16; ++j) {
                            const uint32_t ao = (ky * kTW * C::kRow + 32 * j) / 16;
                            const uint32_t bo = (ky * C::kN * C::kRow + 32 * j) / 16;
                            mma_bf16(d0, ((uint64_t)dhi << 32) | (a_lo + ao),
                                     ((uint64_t)dhi << 32) | (b_lo + bo), idesc,
                                     (q | ky | j) != 0 ? 1u : 0u);
                        }
                    }
                    mma_commit(empty + s);
                }
                mma_commit(tfull + ab);
            }
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        const int eg = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;
        const int tx = m % kTW, ty = m / kTW;  // input pixel of this lane
        const float slope = act_slope(p.act, p.alpha);
        const f32x2 slope2 = f2(slope, slope);
        uint32_t acc = (uint32_t)eg;
        ItemWalk walk;
        walk.init(p, blockIdx.x + eg * gridDim.x, C::kEpiGroups * gridDim.x);
        for (int item = blockIdx.x + eg * gridDim.x; item < p.n_items;
             item += C::kEpiGroups * gridDim.x, acc += C::kEpiGroups, walk.next(p)) {
            const int img = walk.IMG(p), x0 = walk.TX(p) * kKxCols, y0 = (p.ty0 + walk.TY(p)) * kTH;
            const uint32_t ab = acc % C::kAcc, aph = (acc / C::kAcc) & 1u;
            mbar_wait(tfull + ab, aph);
            fence_after_sync();
            const uint32_t tbase = tmem + ab * C::kN + ((uint32_t)(quarter * 32) << 16);
            const int gx = x0 + tx - 1, gy = y0 + ty;
            const bool inner = tx >= 1 && tx <= kKxCols;
            const bool valid = inner && gx < p.w && gy < p.h;
            float hacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            auto release = [&]() {  // item fully read -> hand the TMEM buffer back
                fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + ab);
            };
            // one 16-channel half: kx sum, BN fold, activation, stores / pool / head
            auto half = [&](int h2, const uint32_t(&t0)[16], const uint32_t(&t1)[16],
                            const uint32_t(&t2)[16]) {
                const int n = h2 * 16;
                const float4 *sc4 = reinterpret_cast<const float4 *>(s_scale + n);
                const float4 *sh4 = reinterpret_cast<const float4 *>(s_shift + n);
                float v[16];
#pragma unroll
                for (int i4 = 0; i4 < 4; ++i4) {
                    const float4 sc = sc4[i4], sh = sh4[i4];
                    const f32x2 sc2[2] = {f2(sc.x, sc.y), f2(sc.z, sc.w)};
                    const f32x2 sh2[2] = {f2(sh.x, sh.y), f2(sh.z, sh.w)};
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const int i = 4 * i4 + 2 * jp;
                        // T0 of the left neighbour, T2 of the right one, two channels at a time
                        const f32x2 left =
                            f2(__shfl_up_sync(0xffffffffu, __uint_as_float(t0[i]), 1),
                               __shfl_up_sync(0xffffffffu, __uint_as_float(t0[i + 1]), 1));
                        const f32x2 right =
                            f2(__shfl_down_sync(0xffffffffu, __uint_as_float(t2[i]), 1),
                               __shfl_down_sync(0xffffffffu, __uint_as_float(t2[i + 1]), 1));
                        const f32x2 mid = f2(__uint_as_float(t1[i]), __uint_as_float(t1[i + 1]));
                        const f32x2 d = add2(add2(left, mid), right);
                        act2(fma2(d, sc2[jp], sh2[jp]), slope2, v[i], v[i + 1]);
                    }
                }
                if (MODE == kHead) {
                    head_accumulate(s_hw, p.cout, p.head_c, n, v, hacc);
                    if (!p.y && !p.y_f32) return;
                }
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                if (valid) {
                    const int64_t pix = ((int64_t)img * p.h + gy) * p.w + gx;
                    if (p.y) st_global_v8(p.y + pix * p.cout + n, pk);
                    if (p.y_f32) {
                        float4 *dst = reinterpret_cast<float4 *>(p.y_f32 + pix * p.cout + n);
                        dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                        dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                        dst[2] = make_float4(v[8], v[9], v[10], v[11]);
                        dst[3] = make_float4(v[12], v[13], v[14], v[15]);
                    }
                }
                if (MODE == kPool) {
                    // output column gx = x0 + tx - 1 with x0 even: pairs (tx, tx+1), tx odd;
                    // rows pair as lanes ^16 (ty even / odd in the same warp)
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t a = hmax2u(pk[i], __shfl_down_sync(0xffffffffu, pk[i], 1));
                        pk[i] = hmax2u(a, __shfl_xor_sync(0xffffffffu, a, 16));
                    }
                    if (valid && (tx & 1) && !(ty & 1)) {
                        const int64_t pp = ((int64_t)img * (p.h / 2) + gy / 2) * (p.w / 2) + gx / 2;
                        st_global_v8(p.pool + pp * p.cout + n, pk);
                    }
                }
            };
            if (LS_KX_PIPE && COUT == 32) {
                // both halves' loads in flight before the first half is processed
                uint32_t a0[16], a1[16], a2[16], b0[16], b1[16], b2[16];
                tmem_ld16_async(tbase + 0u, a0);
                tmem_ld16_async(tbase + (uint32_t)COUT, a1);
                tmem_ld16_async(tbase + (uint32_t)(2 * COUT), a2);
                tmem_ld_wait3(a0, a1, a2);
                tmem_ld16_async(tbase + 16u, b0);
                tmem_ld16_async(tbase + (uint32_t)(COUT + 16), b1);
                tmem_ld16_async(tbase + (uint32_t)(2 * COUT + 16), b2);
                half(0, a0, a1, a2);
                tmem_ld_wait3(b0, b1, b2);
                release();
                half(1, b0, b1, b2);
            } else {
#pragma unroll(COUT == 32 ? 2 : 1)
                for (int h2 = 0; h2 < COUT / 16; ++h2) {
                    const int n = h2 * 16;
                    uint32_t t0[16], t1[16], t2[16];
                    tmem_ld16_async(tbase + (uint32_t)(0 * COUT + n), t0);
                    tmem_ld16_async(tbase + (uint32_t)(1 * COUT + n), t1);
                    tmem_ld16_async(tbase + (uint32_t)(2 * COUT + n), t2);
                    tmem_ld_wait3(t0, t1, t2);
                    if (h2 == COUT / 16 - 1) release();
                    half(h2, t0, t1, t2);
                }
            }
            if (MODE == kHead && valid) {
                const int64_t pix = ((int64_t)img * p.h + gy) * p.w + gx;
                for (int j2 = 0; j2 < p.head_c; ++j2) {
                    const float z = hacc[j2] + __ldg(p.head_b + j2);
                    p.head_out[pix * p.head_c + j2] = sigmoid_fast(z);
                }
            }
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
}

// ---------------------------------------------------------------------------
// cout = 32 convolutions over pixel PAIRS (the full-resolution e0c2, d0c1,
// d0c2 + head layers; sources of 32 channels).  The NHWC input is read as
// (W/2) "pair pixels" of 64 channels P(j) = [x(2j), x(2j+1)] (one 128 B
// swizzled operand row), so a 128-row A tile is 8 rows x 16 pairs and TMEM
// lane j holds both outputs of its pair, N = 64 = [out(2j) | out(2j+1)]:
//   MMA_0  (N=64)  A = P(j),   B rows [W(kx=1+e) ; W(kx=e)] for element e
//                  -- every tap whose input and output share the pair
//   MMA_-1 (N=32)  A = P(j-1) element 1 = x(2j-1), B = W(kx=0) -> out(2j)
//   MMA_+1 (N=32)  A = P(j+1) element 0 = x(2j+2), B = W(kx=2) -> out(2j+1)
// MMA_-1 / MMA_+1 address the neighbouring pair through a descriptor start
// one operand row earlier / later (tcgen05 descriptors may start at any row
// of a swizzled tile, scripts/umma_shift_test.cu), so the kx sum happens in
// the tensor core: the epilogue has no cross-lane shuffles and reads 32 TMEM
// columns per output pixel instead of 96 (k_conv_kx).  Lanes of pair columns
// 0 and 15 of a tile row see the wrong neighbour: tiles advance by 14 pairs.
// Weights stay resident, loaded from the ABI's [tap][n][c] layout as
// 16-channel x 32-row boxes into 32 B-swizzled B tiles.
constexpr int kPxCols = 14;  // output pairs per tile row

struct CfgPx {
    static constexpr uint32_t kRow = 128;        // A operand row: 64 bf16 channels
    static constexpr int kN = 64;                // [out(2j) | out(2j+1)] x 32
    static constexpr int kAcc = 7;               // TMEM buffers of 64 columns
    static constexpr int kEpiGroups = 4;
    static constexpr int kThreads = 64 + 128 * kEpiGroups;
    static constexpr int kTmemCols = 512;
    static constexpr uint32_t kBTile = 2048;     // 64 rows x 32 B
    static constexpr uint32_t kRingPad = 1024;   // MMA_-1 of stage 0 reads one row before it
};

// C8: the network's 8-channel input layer (e0c1).  A pair row is then 16
// channels (32 B, 32 B swizzle), one K16 step per ky covers both elements, and
// the three B tiles per ky ([W(1)|W(2)] ; [W(0)|W(1)] for N=64, [0|W(0)] and
// [W(2)|0] for the N=32 neighbour MMAs) mix 8-channel halves of two taps, so
// the epilogue warps assemble them in shared memory (manual 32 B swizzle)
// instead of TMA.
// KX2: pixel pairs WITHOUT neighbour-row MMAs.  Per K16 step two N=96 MMAs
// against ONE B tile [W(2) ; W(1) ; W(0)] (96 rows) write TMEM columns
//   [ spill-left | out(2j) | out(2j+1) | spill-right ]  (4 x 32)
// element 0 (x(2j)) at columns 0..95, element 1 (x(2j+1)) at 32..127, and the
// epilogue adds the neighbours' spills: out(2j) += spill-right of lane j-1,
// out(2j+1) += spill-left of lane j+1.  Same MMA count and operand bytes per
// pixel as k_conv_kx with half its shuffles and 2/3 of its TMEM reads, and no
// row-shifted operands -- for the two-source d0c1, where the neighbour-row
// MMAs' extra operand reads lose.
// epilogue warpgroups: KX2 items hold 128 TMEM columns and their epilogue
// more live registers (three groups: 448 threads, up to 144 registers)
template <bool G3, int CO = 32, bool C8NBR = false>
__host__ __device__ constexpr int px_groups() {
    return C8NBR ? LS_C8_GROUPS
                 : G3 ? (CO == 64 ? LS_KX2_64_GROUPS : LS_KX2_GROUPS) : CfgPx::kEpiGroups;
}

// KX2 with 64 channels (CO = 64 outputs, CI = 32 or 64 inputs; the half-
// resolution enc1 / dec1 layers): TMEM item [spill-left | out(2j) | out(2j+1) |
// spill-right] x 64 = 256 columns (2 buffers), N = 192 MMAs, B tiles of 192 rows.
// With CI = 64 a pair's two pixels are 128 B rows of two TMA boxes (a 5-D view
// [c][element][pair][row][image] of the NHWC tensor, one box per element).
template <int MODE, bool C8, bool KX2 = false, int CO = 32, int CI = 32>
__global__ void __launch_bounds__(64 + 128 * px_groups<KX2 || C8, CO, C8 && !KX2>()) k_conv_px2(
    const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
    const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mY,
    const ConvParamsP p) {
    static_assert(CO == 32 || (!C8 && MODE != kHead), "64-channel pixel pairs: no head");
    static_assert(CI == 32 || (!C8 && CO == 64), "64-channel inputs: 64-channel forms only");
    using C = CfgPx;
    // TMEM columns per item: KX2 [sl | o0 | o1 | sr] x CO, neighbour-row [o0 | o1] x CO
    constexpr int kN = KX2 ? 4 * CO : (C8 ? C::kN : 2 * CO);
    constexpr int kAcc = KX2 ? 512 / kN : (CO == 64 ? 4 : C::kAcc);
    constexpr uint32_t kBTn = 2u * CO * 32u;      // neighbour-row B tile [W(1+e) ; W(e)] bytes
    constexpr int kGroups = px_groups<KX2 || C8, CO, C8 && !KX2>();
    // an epilogue group waits on an accumulator's tfull parity at most one phase
    // ahead only if groups <= buffers (3 groups on 2 buffers read stale items)
    static_assert(!KX2 || kGroups <= kAcc, "KX2: epilogue warpgroups <= TMEM buffers");
    constexpr int kT = CI / 16;                   // K16 steps per element and source
    constexpr uint32_t kBT = 3u * CO * 32u;       // KX2 B tile [W(2) ; W(1) ; W(0)] bytes
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const int S = p.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bar);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + kAcc;
    uint64_t *bres = tempty + kAcc;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bres + 1);
    const int nsrc = p.nq;  // 1 or 2 sources of 32 channels, one 64-channel pair chunk each

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, 1);
            }
            for (int a = 0; a < kAcc; ++a) {
                mbar_init(tfull + a, 1);
                mbar_init(tempty + a, 4);
            }
            mbar_init(bres, 1);
            fence_barrier_init();
            tma_prefetch(&mA0);
            if (nsrc > 1) tma_prefetch(&mA1);
            tma_prefetch(&mB);
        }
        __syncwarp();
        tmem_alloc(tslot, C::kTmemCols);
    } else if (warp >= 2) {
        // (BN constants and head weights are kernel parameters: p.pc_*)
        const int t = threadIdx.x - 64;
        constexpr int kEpiThreads = 128 * kGroups;
        if (C8) {
            // per ky 4 KB: [0, 2 KB) the N=64 tile, [2, 3) [0|W0], [3, 4) [W2|0];
            // one thread per (ky, row, 16 B half); W is [tap][32][16] bf16
            const uint16_t *wg = reinterpret_cast<const uint16_t *>(p.wts);
            for (int i = t; i < 3 * 128 * 2; i += kEpiThreads) {
                const int ky = i / 256, r = (i >> 1) & 127, hf = i & 1;
                int kx = -1, co = r & 31;
                if (KX2) {
                    // one N = 128 tile [spill-left | out(2j) | out(2j+1) | spill-right]
                    // against the pair [x(2j) | x(2j+1)]
                    if (r < 32) kx = hf ? -1 : 2;         // -> out(2j-1): x(2j) with W(2)
                    else if (r < 64) kx = hf ? 2 : 1;     // -> out(2j)
                    else if (r < 96) kx = hf ? 1 : 0;     // -> out(2j+1)
                    else kx = hf ? 0 : -1;                // -> out(2j+2): x(2j+1) with W(0)
                } else if (r < 32) kx = hf ? 2 : 1;   // out(2j)   <- [x(2j) | x(2j+1)]
                else if (r < 64) kx = hf ? 1 : 0;     // out(2j+1) <- [x(2j) | x(2j+1)]
                else if (r < 96) kx = hf ? 0 : -1;    // out(2j)   <- x(2j-1) (element 1)
                else kx = hf ? -1 : 2;                // out(2j+1) <- x(2j+2) (element 0)
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (kx >= 0) v = *reinterpret_cast<const uint4 *>(wg + ((kx * 3 + ky) * 32 + co) * 16);
                const uint32_t a = (uint32_t)(r * 32 + hf * 16);
                *reinterpret_cast<uint4 *>(smem + p.off_b + ky * 4096 + (a ^ (((a >> 7) & 1u) << 4))) = v;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    // B tile (source s, ky, element e, channel block t): rows 0-31 = W(kx=1+e),
    // rows 32-63 = W(kx=e), 16 channels each
    auto btile = [&](int src, int ky, int e, int t) -> uint32_t {
        return p.off_b + (uint32_t)((((src * 3 + ky) * 2 + e) * kT + t)) * kBTn;
    };
    constexpr uint32_t kARow = C8 ? 32u : C::kRow;

    if (warp == 0) {
        if (elect_one()) {
            // ------------------------------ TMA producer ------------------------------
            if (C8) {
                mbar_arrive(bres);  // B tiles were built before the block barrier
            } else if (KX2) {
                // tile (src, ky, t): rows [W(2) ; W(1) ; W(0)], kBT bytes
                mbar_expect_tx(bres, (uint32_t)(nsrc * 3 * kT) * kBT);
                for (int src = 0; src < nsrc; ++src)
                    for (int ky = 0; ky < 3; ++ky)
                        for (int t = 0; t < kT; ++t)
                            for (int r = 0; r < 3; ++r)
                                tma_load_3d(smem + p.off_b + ((src * 3 + ky) * kT + t) * kBT +
                                                r * (CO * 32),
                                            &mB, src * CI + 16 * t, 0, (2 - r) * 3 + ky, bres);
            } else {
                mbar_expect_tx(bres, (uint32_t)(nsrc * 3 * 2 * kT) * kBTn);
            }
            for (int src = 0; src < ((C8 || KX2) ? 0 : nsrc); ++src)
                for (int ky = 0; ky < 3; ++ky)
                    for (int e = 0; e < 2; ++e)
                        for (int t = 0; t < kT; ++t)
                            for (int r = 0; r < 2; ++r) {
                                const int kx = r == 0 ? 1 + e : e;
                                tma_load_3d(smem + btile(src, ky, e, t) + r * (kBTn / 2), &mB,
                                            src * CI + 16 * t, 0, kx * 3 + ky, bres);
                            }
            LS_GDC_WAIT();
            int s = 0;
            uint32_t ph = 0;
            ItemWalk walk;
            walk.init(p, blockIdx.x, gridDim.x);
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, walk.next(p)) {
                const int img = walk.IMG(p), px0 = walk.TX(p) * kPxCols - 1,
                          y0 = (p.ty0 + walk.TY(p)) * kTH;
                for (int q = 0; q < nsrc; ++q, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                    mbar_wait(empty + s, ph ^ 1u);
                    uint8_t *st = smem + C::kRingPad + (size_t)s * p.stage_bytes;
                    if constexpr (CI == 64) {
                        // element 0 / element 1 boxes of the pair-split 5-D view
                        mbar_expect_tx(full + s, 2u * p.a_tx);
                        tma_load_5d(st, q ? &mA1 : &mA0, 0, 0, px0, y0 - 1, img, full + s);
                        tma_load_5d(st + p.a_bytes, q ? &mA1 : &mA0, 0, 1, px0, y0 - 1, img, full + s);
                    } else {
#ifdef LS_EXP_PX_NOTMA  // timing experiment only (scripts/exp): wrong outputs
                        mbar_arrive(full + s);
                        (void)st;
#else
                        mbar_expect_tx(full + s, p.a_tx);
                        tma_load_4d(st, q ? &mA1 : &mA0, 0, px0, y0 - 1, img, full + s);
#endif
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            // ------------------------------- MMA issuer -------------------------------
            const uint32_t id64 = idesc_bf16(128, 64), id32 = idesc_bf16(128, 32);
            // KX2 MMA shapes: 3, 2 and 1 output blocks of CO columns
            const uint32_t idN3 = idesc_bf16(128, 3 * CO), idN2 = idesc_bf16(128, 2 * CO),
                           idN1 = idesc_bf16(128, CO);
            const uint64_t aproto = smem_desc(0, kARow, C8 ? kSwizzle32B : kSwizzle128B);
            const uint64_t bproto = smem_desc(0, 32, kSwizzle32B);
            const uint32_t ahi = (uint32_t)(aproto >> 32), alo = (uint32_t)aproto;
            const uint32_t bhi = (uint32_t)(bproto >> 32), blo = (uint32_t)bproto;
            mbar_wait(bres, 0);
            int s = 0;
            uint32_t ph = 0, ab = 0, aph = 0;
            for (int item = blockIdx.x; item < p.n_items;
                 item += gridDim.x, ab = ab + 1 == kAcc ? 0 : ab + 1, aph ^= ab == 0) {
                mbar_wait(tempty + ab, aph ^ 1u);
                fence_after_sync();
                const uint32_t d0 = tmem + ab * kN;
                for (int q = 0; q < nsrc; ++q, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0) {
                    mbar_wait(full + s, ph);
                    fence_after_sync();
                    const uint32_t a_lo =
                        alo + ((sbase + C::kRingPad + (uint32_t)s * p.stage_bytes) >> 4);
                    const uint32_t b_lo = blo + ((sbase + btile(q, 0, 0, 0)) >> 4);
                    if constexpr (C8 && KX2) {
                        // 8-channel input, spill-column form: ONE N = 128 MMA per ky
                        // (the pair's 16 channels are one K16 step)
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) {
                            const uint32_t ar = (uint32_t)(ky * kTW) * kARow / 16;
                            const uint32_t bt = (uint32_t)ky * 4096 / 16;
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + ar),
                                     ((uint64_t)bhi << 32) | (b_lo + bt), idesc_bf16(128, 128),
                                     ky ? 1u : 0u);
                        }
                    } else if constexpr (KX2) {
                        const uint32_t bk =
                            blo + ((sbase + p.off_b + (uint32_t)q * 3 * kT * kBT) >> 4);
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) {
#pragma unroll
                            for (int t = 0; t < kT; ++t) {
                                const uint32_t arow = (uint32_t)(ky * kTW) * C::kRow;
                                // CI = 32: both elements in one 128 B pair row; CI = 64:
                                // element 1 in the second box of the stage
                                const uint32_t a_e0 = (arow + 32 * t) / 16;
                                const uint32_t a_e1 =
                                    (CI == 64 ? p.a_bytes + arow + 32 * t : arow + 64 + 32 * t) / 16;
                                const uint32_t bt = (uint32_t)((ky * kT + t) * kBT) / 16;
                                const bool first = (q | ky | t) == 0;
                                // element 0 -> [spill-left | out(2j) | out(2j+1)]
                                mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + a_e0),
                                         ((uint64_t)bhi << 32) | (bk + bt), idN3, first ? 0u : 1u);
                                if (first) {
                                    // element 1's first step: columns CO..3CO-1 accumulate onto
                                    // element 0's, 3CO..4CO-1 (spill-right) start fresh
                                    mma_bf16(d0 + CO, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                             ((uint64_t)bhi << 32) | (bk + bt), idN2, 1u);
                                    mma_bf16(d0 + 3 * CO, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                             ((uint64_t)bhi << 32) | (bk + bt + 2 * CO * 32 / 16), idN1,
                                             0u);
                                } else {
                                    // element 1 -> [out(2j) | out(2j+1) | spill-right]
                                    mma_bf16(d0 + CO, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                             ((uint64_t)bhi << 32) | (bk + bt), idN3, 1u);
                                }
                            }
                        }
                    } else if constexpr (C8) {
#pragma unroll
                        for (int ky = 0; ky < LS_EXP_PX_C8_KY; ++ky) {
                            const uint32_t ar = (uint32_t)(ky * kTW) * kARow / 16;
                            const uint32_t bt = (uint32_t)ky * 4096 / 16;
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + ar),
                                     ((uint64_t)bhi << 32) | (b_lo + bt), id64, ky ? 1u : 0u);
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + ar - kARow / 16),
                                     ((uint64_t)bhi << 32) | (b_lo + bt + 2048 / 16), id32, 1u);
                            mma_bf16(d0 + 32, ((uint64_t)ahi << 32) | (a_lo + ar + kARow / 16),
                                     ((uint64_t)bhi << 32) | (b_lo + bt + 3072 / 16), id32, 1u);
                        }
                    } else {
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
#pragma unroll
                        for (int t = 0; t < kT; ++t) {
                            // A: operand row (ky*16 + pair), K offset e*64 B + t*32 B
                            // (64-channel inputs: element e in box e of the stage)
                            const uint32_t arow = (uint32_t)(ky * kTW) * C::kRow;
                            const uint32_t a_e0 = (arow + 32 * t) / 16;
                            const uint32_t a_e1 =
                                (CI == 64 ? p.a_bytes + arow + 32 * t : arow + 64 + 32 * t) / 16;
                            const uint32_t b_e0 = ((ky * 2 + 0) * kT + t) * kBTn / 16;
                            const uint32_t b_e1 = ((ky * 2 + 1) * kT + t) * kBTn / 16;
                            const uint32_t first = (q | ky | t) == 0 ? 0u : 1u;
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + a_e0),
                                     ((uint64_t)bhi << 32) | (b_lo + b_e0), idN2, first);
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                     ((uint64_t)bhi << 32) | (b_lo + b_e1), idN2, 1u);
                            // x(2j-1) -> out(2j): previous row's element 1, W(kx=0)
                            mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + a_e1 - C::kRow / 16),
                                     ((uint64_t)bhi << 32) | (b_lo + b_e0 + kBTn / 32), idN1, 1u);
                            // x(2j+2) -> out(2j+1): next row's element 0, W(kx=2)
                            mma_bf16(d0 + CO, ((uint64_t)ahi << 32) | (a_lo + a_e0 + C::kRow / 16),
                                     ((uint64_t)bhi << 32) | (b_lo + b_e1), idN1, 1u);
                        }
                    }
                    }
                    mma_commit(empty + s);
                }
                mma_commit(tfull + ab);
            }
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        const int eg = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;
        const int tp = m % kTW, ty = m / kTW;  // pair column / row of this lane
        const float slope = act_slope(p.act, p.alpha);
        const f32x2 slope2 = f2(slope, slope);
        const int wp = p.w >> 1;
        uint32_t ab = (uint32_t)eg % kAcc, aph = ((uint32_t)eg / kAcc) & 1u;
        // staging buffer of this warp and item (p.stage_store buffers per warp, used
        // in turn): free once the store that last read it is done reading
        uint32_t sbuf = (uint32_t)(warp - 2) * (uint32_t)p.stage_store;
        ItemWalk walk;
        walk.init(p, blockIdx.x + eg * gridDim.x, kGroups * gridDim.x);
        for (int item = blockIdx.x + eg * gridDim.x; item < p.n_items;
             item += kGroups * gridDim.x, walk.next(p)) {
            const int img = walk.IMG(p), px0 = walk.TX(p) * kPxCols - 1, y0 = (p.ty0 + walk.TY(p)) * kTH;
            mbar_wait(tfull + ab, aph);
            fence_after_sync();
            if (CO == 32 && p.stage_store) {
                if (lane == 0) {
                    if (p.stage_store == 2) tma_store_wait_read_1();
                    else tma_store_wait_read();
                }
                __syncwarp();
            }
            const uint32_t tbase = tmem + ab * kN + ((uint32_t)(quarter * 32) << 16);
            const int gp = px0 + tp, gy = y0 + ty;
            const bool valid = tp >= 1 && tp <= kPxCols && gp < wp && gy < p.h;
            // this lane's first output pixel and the item's store bases (one 64-bit
            // address computation per item instead of one per 16-channel store)
            const int64_t pix0 = ((int64_t)img * p.h + gy) * p.w + 2 * gp;
            __nv_bfloat16 *const ybase = p.y ? p.y + pix0 * CO : nullptr;
            __nv_bfloat16 *const pbase =
                MODE == kPool ? p.pool + (((int64_t)img * (p.h / 2) + gy / 2) * (p.w / 2) + gp) * CO
                              : nullptr;
            // head sums per pixel and output as {even channels, odd channels}
            // partials: the activations come out of the packed epilogue math as
            // channel pairs, so each FFMA2 takes them as they are
            f32x2 hsum[2][4] = {{0ull, 0ull, 0ull, 0ull}, {0ull, 0ull, 0ull, 0ull}};
            uint32_t keep[8];  // pixel 2j's packed half for the horizontal pool
            // 16-column groups in the order (px0, ch 0-15), (px1, 0-15), (px0, 16-31),
            // (px1, 16-31); group g+1's tcgen05.ld is in flight while g is processed
            uint32_t ra[16], rb[16];
            auto col = [&](int g) -> uint32_t { return tbase + (uint32_t)((g & 1) * CO + (g >> 1) * 16); };
            // BN fold + activation of 16 channels of NP pixels (constants read once)
            auto bnact = [&](int n, const uint32_t(&r0)[16], const uint32_t(&r1)[16],
                             float(&v0)[16], float(&v1)[16], int np) {
#pragma unroll
                for (int i4 = 0; i4 < 4; ++i4) {
                    const float *sc = p.pc_scale + n + 4 * i4;
                    const float *sh = p.pc_shift + n + 4 * i4;
                    const f32x2 sc2[2] = {f2(sc[0], sc[1]), f2(sc[2], sc[3])};
                    const f32x2 sh2[2] = {f2(sh[0], sh[1]), f2(sh[2], sh[3])};
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const int i = 4 * i4 + 2 * jp;
                        act2(fma2(f2(__uint_as_float(r0[i]), __uint_as_float(r0[i + 1])), sc2[jp],
                                  sh2[jp]),
                             slope2, v0[i], v0[i + 1]);
                        if (np > 1)
                            act2(fma2(f2(__uint_as_float(r1[i]), __uint_as_float(r1[i + 1])),
                                      sc2[jp], sh2[jp]),
                                 slope2, v1[i], v1[i + 1]);
                    }
                }
            };
            // head / bf16 stores / pool of one pixel's 16 channels
            auto emit = [&](int g, const float(&v)[16]) {
                const int px = g & 1, n = (g >> 1) * 16;
                if (MODE == kHead) {
                    // one FFMA2 per channel pair and head output (weights from the
                    // constant bank as pairs)
#pragma unroll
                    for (int j2 = 0; j2 < 4; ++j2) {
                        if (j2 >= p.head_c) break;
                        const float *wp = p.pc_head + j2 * 32 + n;
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            hsum[px][j2] = fma2(f2(wp[2 * i], wp[2 * i + 1]),
                                                f2(v[2 * i], v[2 * i + 1]), hsum[px][j2]);
                    }
                    if (!p.y && !p.y_f32) return;
                }
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                if (CO == 32 && p.stage_store) {
                    // staging row (tile row parity, pair - 1): the pair's 2 x 32
                    // channels, 16 B chunks XOR-swizzled by row (TMA 128 B)
                    if (valid) {
                        const int r = (ty & 1) * kPxCols + tp - 1, c = px * 4 + (n >> 3);
                        uint8_t *row = smem + p.off_stage + sbuf * 4096u + r * 128;
                        *reinterpret_cast<uint4 *>(row + ((c ^ (r & 7)) << 4)) =
                            make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        *reinterpret_cast<uint4 *>(row + (((c + 1) ^ (r & 7)) << 4)) =
                            make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    }
                } else if (valid LS_EXP_PX_STORE_GUARD) {
                    // element offsets from the item's per-lane base (cout = CO)
                    if (p.y) st_global_v8(ybase + px * CO + n, pk);
                    if (p.y_f32) {
                        const int64_t pix = pix0 + px;
                        float4 *dst = reinterpret_cast<float4 *>(p.y_f32 + pix * p.cout + n);
                        dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                        dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                        dst[2] = make_float4(v[8], v[9], v[10], v[11]);
                        dst[3] = make_float4(v[12], v[13], v[14], v[15]);
                    }
                }
                if (MODE == kPool) {
                    if (px == 0) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) keep[i] = pk[i];
                    } else {
                        // horizontal partner in-lane, vertical partner 16 lanes away
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const uint32_t a = hmax2u(keep[i], pk[i]);
                            pk[i] = hmax2u(a, __shfl_xor_sync(0xffffffffu, a, 16));
                        }
                        if (valid && !(ty & 1)) st_global_v8(pbase + n, pk);
                    }
                }
            };
            auto process = [&](int g, const uint32_t(&rr)[16]) {
                float v[16];
                bnact((g >> 1) * 16, rr, rr, v, v, 1);
                emit(g, v);
            };
            if constexpr (KX2) {
                // 16-channel block n: out(2j) = own + left lane's spill-right,
                // out(2j+1) = own + right lane's spill-left
#pragma unroll
                for (int h2 = 0; h2 < CO / 16; ++h2) {
                    const uint32_t n = 16u * h2;
                    uint32_t sl[16], o0[16], o1[16], sr[16];
                    tmem_ld16_async(tbase + n, sl);
                    tmem_ld16_async(tbase + (uint32_t)CO + n, o0);
                    tmem_ld16_async(tbase + (uint32_t)(2 * CO) + n, o1);
                    tmem_ld16_async(tbase + (uint32_t)(3 * CO) + n, sr);
                    tmem_ld_wait4(sl, o0, o1, sr);
                    if (h2 == CO / 16 - 1) {  // item fully read -> hand the TMEM buffer back
                        fence_before_sync();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(tempty + ab);
                    }
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        // two channels per FADD2 (same IEEE adds as the scalar form)
                        float a0, a1, b0, b1;
                        unf2(add2(f2(__uint_as_float(o0[i]), __uint_as_float(o0[i + 1])),
                                  f2(__shfl_up_sync(0xffffffffu, __uint_as_float(sr[i]), 1),
                                     __shfl_up_sync(0xffffffffu, __uint_as_float(sr[i + 1]), 1))),
                             a0, a1);
                        unf2(add2(f2(__uint_as_float(o1[i]), __uint_as_float(o1[i + 1])),
                                  f2(__shfl_down_sync(0xffffffffu, __uint_as_float(sl[i]), 1),
                                     __shfl_down_sync(0xffffffffu, __uint_as_float(sl[i + 1]), 1))),
                             b0, b1);
                        o0[i] = __float_as_uint(a0);
                        o0[i + 1] = __float_as_uint(a1);
                        o1[i] = __float_as_uint(b0);
                        o1[i + 1] = __float_as_uint(b1);
                    }
                    float v0[16], v1[16];
                    bnact((int)n, o0, o1, v0, v1, 2);
                    emit(2 * h2, v0);
                    emit(2 * h2 + 1, v1);
                }
            } else {
            // both pixels of a 16-channel block per step (BN constants read once);
            // the next block's loads are in flight while one is processed
            uint32_t rc[16], rd[16];
            tmem_ld16_async(col(0), ra);
            tmem_ld16_async(col(1), rb);
            tmem_ld_wait16(ra);
            tmem_ld_wait16(rb);
#pragma unroll
            for (int blk = 0; blk < CO / 16; ++blk) {
                // (blocks alternate between the (ra, rb) and (rc, rd) registers)
                uint32_t(&c0)[16] = (blk & 1) ? rc : ra;
                uint32_t(&c1)[16] = (blk & 1) ? rd : rb;
                uint32_t(&n0)[16] = (blk & 1) ? ra : rc;
                uint32_t(&n1)[16] = (blk & 1) ? rb : rd;
                if (blk + 1 < CO / 16) {
                    tmem_ld16_async(col(2 * blk + 2), n0);
                    tmem_ld16_async(col(2 * blk + 3), n1);
                } else {
                    // item fully read -> hand the TMEM buffer back
                    fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty + ab);
                }
                float v0[16], v1[16];
                bnact(16 * blk, c0, c1, v0, v1, 2);
                emit(2 * blk, v0);
                emit(2 * blk + 1, v1);
                if (blk + 1 < CO / 16) {
                    tmem_ld_wait16(n0);
                    tmem_ld_wait16(n1);
                }
            }
            }
            if (CO == 32 && p.stage_store) {
                // the warp's two tile rows x 14 pairs: one TMA store (clipped at the
                // image's right / bottom edge)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    tma_store_4d(&mY, smem + p.off_stage + sbuf * 4096u, 0, px0 + 1,
                                 y0 + 2 * quarter, img);
                if (p.stage_store == 2) sbuf ^= 1u;
            }
            if (MODE == kHead && valid) {
                const int64_t pix = ((int64_t)img * p.h + gy) * p.w + 2 * gp;
                if (p.head_c == 3) {
                    // the pair's 6 outputs are contiguous (pix even): 3 x 8 B stores
                    float o[6];
#pragma unroll
                    for (int j2 = 0; j2 < 3; ++j2) {
                        float e0, o0, e1, o1;
                        unf2(hsum[0][j2], e0, o0);
                        unf2(hsum[1][j2], e1, o1);
                        const float b = __ldg(p.head_b + j2);
                        o[j2] = sigmoid_fast((e0 + o0) + b);
                        o[3 + j2] = sigmoid_fast((e1 + o1) + b);
                    }
                    float2 *dst = reinterpret_cast<float2 *>(p.head_out + pix * 3);
                    dst[0] = make_float2(o[0], o[1]);
                    dst[1] = make_float2(o[2], o[3]);
                    dst[2] = make_float2(o[4], o[5]);
                } else {
#pragma unroll
                    for (int j2 = 0; j2 < 4; ++j2) {
                        if (j2 >= p.head_c) break;
                        float e0, o0, e1, o1;
                        unf2(hsum[0][j2], e0, o0);
                        unf2(hsum[1][j2], e1, o1);
                        const float b = __ldg(p.head_b + j2);
                        p.head_out[pix * p.head_c + j2] = sigmoid_fast((e0 + o0) + b);
                        p.head_out[(pix + 1) * p.head_c + j2] = sigmoid_fast((e1 + o1) + b);
                    }
                }
            }
            // next item of this group: kEpiGroups buffers further on
#pragma unroll 1
            for (int k = 0; k < kGroups; ++k) {
                ab = ab + 1 == kAcc ? 0 : ab + 1;
                aph ^= ab == 0;
            }
        }
    }
    if (CO == 32 && p.stage_store && warp >= 2 && lane == 0)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
}

// ---------------------------------------------------------------------------
// dec0_up fused into dec0_conv1 (FE:model/unet.ts:170-181: upsample, concat
// [up, skip], conv1).  Per item the 2x2 transposed conv of the half-resolution
// dec1 output runs on the tensor core (M = 128 half-resolution pixels of an
// 8-row x 16-column box, N = 128 = (dy, dx, co), K = 64), and a transform
// warpgroup adds its bias, rounds to bf16 -- the values the unfused up tensor
// would hold -- and writes them pixel-shuffled straight into the KX2 A operand
// of source 0 (10 rows x 16 pairs x 128 B, 128 B swizzle), zero outside the
// image (the conv's "same" padding of the up tensor).  The 134 MB up tensor is
// neither written nor read.  Source 1 (skip) and the epilogue are the KX2
// form's; per item the MMA thread issues skip's MMAs, then the next item's up
// MMAs, then source 0's, so the transform overlaps tensor work.
// Ring order per item: [dec1 box, skip box]; TMEM columns 0..383 hold three
// 128-column KX2 accumulators, 384..511 the up accumulator.
// epilogue warpgroups and transform warpgroups (1: all four (dy, dx) blocks; 2:
// one dy each) -- A/B build switches
#ifndef LS_UPF_EPI
#define LS_UPF_EPI 2
#endif
#ifndef LS_UPF_XF
#define LS_UPF_XF 2
#endif
constexpr int kUpGroups = LS_UPF_EPI, kUpXf = LS_UPF_XF;
constexpr uint32_t kUpBox = 10u * 16u * 128u;  // source-0 A box (20 KB)

__global__ void __launch_bounds__(64 + 128 * (kUpGroups + kUpXf)) k_conv_upfuse(
    const __grid_constant__ CUtensorMap mD1, const __grid_constant__ CUtensorMap mSkip,
    const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mU,
    const __grid_constant__ CUtensorMap mY, const ConvParamsP p) {
    using C = CfgPx;
    constexpr int kN = 128, kAcc = 3, kGroups = kUpGroups;
    constexpr uint32_t kUpCol = 384;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const int S = p.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bar);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + kAcc;
    uint64_t *bres = tempty + kAcc;
    uint64_t *upready = bres + 1, *upfree = upready + 1;
    uint64_t *a0ready = upfree + 1, *a0free = a0ready + 2;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(a0free + 2);
    uint8_t *abox = smem + p.off_stage;  // two source-0 A boxes

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, 1);
            }
            for (int a = 0; a < kAcc; ++a) {
                mbar_init(tfull + a, 1);
                mbar_init(tempty + a, 4);
            }
            mbar_init(bres, 1);
            mbar_init(upready, 1);
            mbar_init(upfree, 4 * kUpXf);
            for (int k = 0; k < 2; ++k) {
                mbar_init(a0ready + k, 4 * kUpXf);
                mbar_init(a0free + k, 1);
            }
            fence_barrier_init();
            tma_prefetch(&mD1);
            tma_prefetch(&mSkip);
            tma_prefetch(&mB);
            tma_prefetch(&mU);
        }
        __syncwarp();
        tmem_alloc(tslot, C::kTmemCols);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (elect_one()) {
            // ------------------------------ TMA producer ------------------------------
            // resident: d0c1 KX2 tiles (src, ky, t) [W(2) ; W(1) ; W(0)] and the
            // up weights [(dy, dx, co) = 128 rows][64 channels]
            mbar_expect_tx(bres, 12u * 3072u + 16384u);
            for (int src = 0; src < 2; ++src)
                for (int ky = 0; ky < 3; ++ky)
                    for (int t = 0; t < 2; ++t)
                        for (int r = 0; r < 3; ++r)
                            tma_load_3d(smem + p.off_b + ((src * 3 + ky) * 2 + t) * 3072 + r * 1024,
                                        &mB, src * 32 + 16 * t, 0, (2 - r) * 3 + ky, bres);
            tma_load_3d(smem + p.off_b + 12 * 3072, &mU, 0, 0, 0, bres);
            LS_GDC_WAIT();
            int s = 0;
            uint32_t ph = 0;
            ItemWalk walk;
            walk.init(p, blockIdx.x, gridDim.x);
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, walk.next(p)) {
                const int img = walk.IMG(p), px0 = walk.TX(p) * kPxCols - 1,
                          y0 = (p.ty0 + walk.TY(p)) * kTH;
                // dec1 rows y0/2 - 1 .. y0/2 + 6 (the up rows y0 - 1 .. y0 + 8 come
                // from y0/2 - 1 .. y0/2 + 4), columns px0 .. px0 + 15
                mbar_wait(empty + s, ph ^ 1u);
                mbar_expect_tx(full + s, 16384u);
                tma_load_4d(smem + C::kRingPad + (size_t)s * p.stage_bytes, &mD1, 0, px0, y0 / 2 - 1,
                            img, full + s);
                s = s + 1 == S ? 0 : s + 1;
                ph ^= s == 0;
                mbar_wait(empty + s, ph ^ 1u);
                mbar_expect_tx(full + s, p.a_tx);
                tma_load_4d(smem + C::kRingPad + (size_t)s * p.stage_bytes, &mSkip, 0, px0, y0 - 1,
                            img, full + s);
                s = s + 1 == S ? 0 : s + 1;
                ph ^= s == 0;
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            // ------------------------------- MMA issuer -------------------------------
            const uint32_t id64 = idesc_bf16(128, 64), id32 = idesc_bf16(128, 32);
            const uint32_t id96 = idesc_bf16(128, 96), id128 = idesc_bf16(128, 128);
            const uint64_t a128 = smem_desc(0, 128, kSwizzle128B);
            const uint64_t b32 = smem_desc(0, 32, kSwizzle32B);
            const uint32_t ahi = (uint32_t)(a128 >> 32), alo = (uint32_t)a128;
            const uint32_t bhi = (uint32_t)(b32 >> 32), blo = (uint32_t)b32;
            mbar_wait(bres, 0);
            // ring slot q of the CTA's sequence: item n's dec1 box is slot 2n, its
            // skip box slot 2n + 1 (the producer's order); slots are consumed
            // slightly out of order (the next item's dec1 box before this item's
            // skip box), so stage and phase come from the slot index
            auto stage_of = [&](int q) { return q % S; };
            auto phase_of = [&](int q) { return (uint32_t)(q / S) & 1u; };
            uint32_t upph = 0;
            // up MMAs of item n (dec1 box in slot 2n)
            auto up_mma = [&](int n) {
                const int st = stage_of(2 * n);
                mbar_wait(full + st, phase_of(2 * n));
                fence_after_sync();
                const uint32_t a_lo = alo + ((sbase + C::kRingPad + (uint32_t)st * p.stage_bytes) >> 4);
                const uint32_t b_lo = alo + ((sbase + p.off_b + 12u * 3072u) >> 4);
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    mma_bf16(tmem + kUpCol, ((uint64_t)ahi << 32) | (a_lo + 2u * t),
                             ((uint64_t)ahi << 32) | (b_lo + 2u * t), id128, t ? 1u : 0u);
                mma_commit(empty + st);
                mma_commit(upready);
            };
            // KX2 MMAs of one source (A at a_lo, B tiles of source src); first:
            // the accumulator's first K step
            auto kx2_mma = [&](uint32_t d0, uint32_t a_lo, int src, bool first_src) {
                const uint32_t bk = blo + ((sbase + p.off_b + (uint32_t)src * 6u * 3072u) >> 4);
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) {
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const uint32_t arow = (uint32_t)(ky * kTW) * 128u;
                        const uint32_t a_e0 = (arow + 32 * t) / 16, a_e1 = (arow + 64 + 32 * t) / 16;
                        const uint32_t bt = (uint32_t)((ky * 2 + t) * 3072) / 16;
                        const bool first = first_src && (ky | t) == 0;
                        mma_bf16(d0, ((uint64_t)ahi << 32) | (a_lo + a_e0),
                                 ((uint64_t)bhi << 32) | (bk + bt), id96, first ? 0u : 1u);
                        if (first) {
                            mma_bf16(d0 + 32, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                     ((uint64_t)bhi << 32) | (bk + bt), id64, 1u);
                            mma_bf16(d0 + 96, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                     ((uint64_t)bhi << 32) | (bk + bt + 2048 / 16), id32, 0u);
                        } else {
                            mma_bf16(d0 + 32, ((uint64_t)ahi << 32) | (a_lo + a_e1),
                                     ((uint64_t)bhi << 32) | (bk + bt), id96, 1u);
                        }
                    }
                }
            };
            uint32_t ab = 0, aph = 0;
            int n = 0;
            if ((int)blockIdx.x < p.n_items) up_mma(0);
            for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, ++n,
                     ab = ab + 1 == kAcc ? 0 : ab + 1, aph ^= ab == 0) {
                mbar_wait(tempty + ab, aph ^ 1u);
                fence_after_sync();
                const uint32_t d0 = tmem + ab * kN;
                // the next item's up MMAs once the transform has read this item's
                if (item + (int)gridDim.x < p.n_items) {
                    mbar_wait(upfree, upph);
                    upph ^= 1u;
                    fence_after_sync();
                    up_mma(n + 1);
                }
                // source 0 from the transform's box first (the unfused layer's K
                // order: [up, skip]), then source 1 (skip) from slot 2n + 1
                const int k = n & 1;
                mbar_wait(a0ready + k, (uint32_t)(n >> 1) & 1u);
                fence_after_sync();
                kx2_mma(d0, alo + ((sbase + p.off_stage + (uint32_t)k * kUpBox) >> 4), 0, true);
                mma_commit(a0free + k);
                const int st = stage_of(2 * n + 1);
                mbar_wait(full + st, phase_of(2 * n + 1));
                fence_after_sync();
                kx2_mma(d0, alo + ((sbase + C::kRingPad + (uint32_t)st * p.stage_bytes) >> 4), 1, false);
                mma_commit(empty + st);
                mma_commit(tfull + ab);
            }
        }
    } else if (warp >= 2 + 4 * kGroups) {
        // ------------------------------ up transform ------------------------------
        const int quarter = warp & 3;
        const int xg = (warp - 2 - 4 * kGroups) >> 2;  // transform group: dy blocks
        const int l = quarter * 32 + lane;  // dec1 pixel (r, j) of the item's 8 x 16 box
        const int r = l >> 4, j = l & 15;
        const int wp = p.w >> 1;
        uint32_t upph = 0;
        int n = 0;
        ItemWalk walk;
        walk.init(p, blockIdx.x, gridDim.x);
        for (int item = blockIdx.x; item < p.n_items; item += gridDim.x, walk.next(p), ++n) {
            const int px0 = walk.TX(p) * kPxCols - 1, y0 = (p.ty0 + walk.TY(p)) * kTH;
            const int k = n & 1;
            mbar_wait(upready, upph);
            upph ^= 1u;
            fence_after_sync();
            // (dy, dx) blocks of 32 columns; this buffer k was last read by the
            // MMAs of item n - 2
            mbar_wait(a0free + k, ((uint32_t)(n >> 1) & 1u) ^ 1u);
            const uint32_t tb = tmem + kUpCol + ((uint32_t)(quarter * 32) << 16);
            uint8_t *box = abox + k * kUpBox;
            const bool colok = px0 + j >= 0 && px0 + j < wp;
            uint32_t ra[32], rb[32];
            constexpr int kDd = 4 / kUpXf;     // (dy, dx) blocks per group
            const int dd0 = xg * kDd;
            tmem_ld32_async(tb + 32u * dd0, ra);
#pragma unroll
            for (int di = 0; di < kDd; ++di) {
                const int dd = dd0 + di;
                uint32_t(&cur)[32] = (di & 1) ? rb : ra;
                uint32_t(&nxt)[32] = (di & 1) ? ra : rb;
                tmem_ld_wait(cur);
                if (di + 1 < kDd) {
                    tmem_ld32_async(tb + 32u * (dd + 1), nxt);
                } else {
                    fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(upfree);
                }
                const int dy = dd >> 1, dx = dd & 1;
                const int b = 2 * r + dy - 1;  // box row (up row y0 - 1 + b)
                if (b < 0 || b > 9) continue;
                const int y = y0 - 1 + b;
                const bool zero = !colok || y < 0 || y >= p.h;
                const int row = b * 16 + j;
                uint8_t *rp = box + row * 128;
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8) {  // 8 channels per 16 B chunk
                    uint32_t w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = c8 * 8 + 2 * q;
                        const float v0 = zero ? 0.0f : __uint_as_float(cur[c]) + p.pc_upb[c];
                        const float v1 = zero ? 0.0f : __uint_as_float(cur[c + 1]) + p.pc_upb[c + 1];
                        w[q] = pack_bf16(v0, v1);
                    }
                    const int chunk = dx * 4 + c8;
                    *reinterpret_cast<uint4 *>(rp + ((chunk ^ (row & 7)) << 4)) =
                        make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(a0ready + k);
        }
    } else {
        // --------------------------------- epilogue ---------------------------------
        const int eg = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;
        const int tp = m % kTW, ty = m / kTW;
        const float slope = act_slope(p.act, p.alpha);
        const f32x2 slope2 = f2(slope, slope);
        const int wp = p.w >> 1;
        uint32_t ab = (uint32_t)eg % kAcc, aph = ((uint32_t)eg / kAcc) & 1u;
        ItemWalk walk;
        walk.init(p, blockIdx.x + eg * gridDim.x, kGroups * gridDim.x);
        for (int item = blockIdx.x + eg * gridDim.x; item < p.n_items;
             item += kGroups * gridDim.x, walk.next(p)) {
            const int img = walk.IMG(p), px0 = walk.TX(p) * kPxCols - 1,
                      y0 = (p.ty0 + walk.TY(p)) * kTH;
            mbar_wait(tfull + ab, aph);
            fence_after_sync();
            // staged output (as k_conv_px2): this warp's 4 KB buffer at p.off_pool
            uint8_t *const ybuf = smem + p.off_pool + (uint32_t)(warp - 2) * 4096u;
            if (p.stage_store) {
                if (lane == 0) tma_store_wait_read();
                __syncwarp();
            }
            const uint32_t tbase = tmem + ab * kN + ((uint32_t)(quarter * 32) << 16);
            const int gp = px0 + tp, gy = y0 + ty;
            const bool valid = tp >= 1 && tp <= kPxCols && gp < wp && gy < p.h;
            const int64_t pix0 = ((int64_t)img * p.h + gy) * p.w + 2 * gp;
            __nv_bfloat16 *const ybase = p.y + pix0 * 32;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const uint32_t n = 16u * h2;
                uint32_t sl[16], o0[16], o1[16], sr[16];
                tmem_ld16_async(tbase + n, sl);
                tmem_ld16_async(tbase + 32u + n, o0);
                tmem_ld16_async(tbase + 64u + n, o1);
                tmem_ld16_async(tbase + 96u + n, sr);
                tmem_ld_wait4(sl, o0, o1, sr);
                if (h2 == 1) {
                    fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty + ab);
                }
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    float a0, a1, b0, b1;
                    unf2(add2(f2(__uint_as_float(o0[i]), __uint_as_float(o0[i + 1])),
                              f2(__shfl_up_sync(0xffffffffu, __uint_as_float(sr[i]), 1),
                                 __shfl_up_sync(0xffffffffu, __uint_as_float(sr[i + 1]), 1))),
                         a0, a1);
                    unf2(add2(f2(__uint_as_float(o1[i]), __uint_as_float(o1[i + 1])),
                              f2(__shfl_down_sync(0xffffffffu, __uint_as_float(sl[i]), 1),
                                 __shfl_down_sync(0xffffffffu, __uint_as_float(sl[i + 1]), 1))),
                         b0, b1);
                    o0[i] = __float_as_uint(a0);
                    o0[i + 1] = __float_as_uint(a1);
                    o1[i] = __float_as_uint(b0);
                    o1[i + 1] = __float_as_uint(b1);
                }
#pragma unroll
                for (int px = 0; px < 2; ++px) {
                    const uint32_t(&rr)[16] = px ? o1 : o0;
                    float v[16];
#pragma unroll
                    for (int i4 = 0; i4 < 4; ++i4) {
                        const float *sc = p.pc_scale + n + 4 * i4;
                        const float *sh = p.pc_shift + n + 4 * i4;
                        const f32x2 sc2[2] = {f2(sc[0], sc[1]), f2(sc[2], sc[3])};
                        const f32x2 sh2[2] = {f2(sh[0], sh[1]), f2(sh[2], sh[3])};
#pragma unroll
                        for (int jp = 0; jp < 2; ++jp) {
                            const int i = 4 * i4 + 2 * jp;
                            act2(fma2(f2(__uint_as_float(rr[i]), __uint_as_float(rr[i + 1])), sc2[jp],
                                      sh2[jp]),
                                 slope2, v[i], v[i + 1]);
                        }
                    }
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                    if (p.stage_store) {
                        if (valid) {
                            const int r = (ty & 1) * kPxCols + tp - 1, c = px * 4 + (int)(n >> 3);
                            uint8_t *row = ybuf + r * 128;
                            *reinterpret_cast<uint4 *>(row + ((c ^ (r & 7)) << 4)) =
                                make_uint4(pk[0], pk[1], pk[2], pk[3]);
                            *reinterpret_cast<uint4 *>(row + (((c + 1) ^ (r & 7)) << 4)) =
                                make_uint4(pk[4], pk[5], pk[6], pk[7]);
                        }
                    } else if (valid) {
                        st_global_v8(ybase + px * 32 + n, pk);
                    }
                }
            }
            if (p.stage_store) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) tma_store_4d(&mY, ybuf, 0, px0 + 1, y0 + 2 * quarter, img);
            }
#pragma unroll 1
            for (int kk = 0; kk < kGroups; ++kk) {
                ab = ab + 1 == kAcc ? 0 : ab + 1;
                aph ^= ab == 0;
            }
        }
        if (p.stage_store && lane == 0)
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
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
    // function-local static: initialised once, thread-safe (C++11 magic statics)
    static const EncodeTiledFn fn = [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(ptr);
        return EncodeTiledFn(nullptr);
    }();
    return fn;
}

static CUtensorMapSwizzle swizzle_for(int row_bytes) {
    return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// activations NHWC bf16, box {chunk, 16 columns, box_h rows, 1}
static bool encode_act(CUtensorMap *map, const void *base, int c, int w, int h, int batch,
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

// 64-channel NHWC activations as pixel pairs split by element: a 5-D view
// [c = 64][element = 2][pair = w/2][row][image], box {64, 1, 16, box_h, 1}
// (one 128 B operand row per pair and element, 128 B swizzle)
static bool encode_act_pairsplit(CUtensorMap *map, const void *base, int w, int h, int batch,
                                 int box_h) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[5] = {64, 2, (cuuint64_t)(w / 2), (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[4] = {128, 256, (cuuint64_t)w * 128, (cuuint64_t)h * w * 128};
    cuuint32_t box[5] = {64, 1, (cuuint32_t)kTW, (cuuint32_t)box_h, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// weights [taps][n_total][ctot], box {chunk, bn, kys}
static bool encode_wts(CUtensorMap *map, const void *base, int ctot, int n_total, int taps,
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

// Output of a transposed conv with 32 channels viewed as [n][i][dy][j][dx*32+c]
// (i, j = input pixel; the output pixel is (2i+dy, 2j+dx)), box {64, 16, 2, 8, 1}
// = one 8x16-input-pixel item's 16x32-pixel output tile, 128 B swizzle.
static bool encode_up_store(CUtensorMap *map, void *base, int w_in, int h_in, int batch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t row = (cuuint64_t)2 * w_in * 64;  // one output row, bytes
    cuuint64_t dims[5] = {64, (cuuint64_t)w_in, 2, (cuuint64_t)h_in, (cuuint64_t)batch};
    cuuint64_t strides[4] = {128, row, 2 * row, (cuuint64_t)2 * h_in * row};
    cuuint32_t box[5] = {64, (cuuint32_t)kTW, 2, (cuuint32_t)kTH, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output of a transposed conv with 64 channels as [c][dx][j][dy][image*h_in + i]
// (output pixel (2i+dy, 2j+dx)), box {64, 2, 16, 1, 8}: one 8x16-input-pixel
// item's output rows of one parity dy (= its 128-column n-tile), 128 B swizzle.
static bool encode_up_store64(CUtensorMap *map, void *base, int w_in, int h_in, int batch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t row = (cuuint64_t)2 * w_in * 128;  // one output row, bytes
    cuuint64_t dims[5] = {64, 2, (cuuint64_t)w_in, 2, (cuuint64_t)batch * h_in};
    cuuint64_t strides[4] = {128, 256, row, 2 * row};
    cuuint32_t box[5] = {64, 2, (cuuint32_t)kTW, 1, (cuuint32_t)kTH};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 32-channel NHWC output viewed as [pair: 2 x 32 channels][w/2][h][image], box
// {64, 14, 2, 1}: one epilogue warp's two tile rows of 14 output pairs, 128 B swizzle.
static bool encode_pair_store(CUtensorMap *map, void *base, int w, int h, int batch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t row = (cuuint64_t)w * 64;  // one row, bytes
    cuuint64_t dims[4] = {64, (cuuint64_t)(w / 2), (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[3] = {128, row, (cuuint64_t)h * row};
    cuuint32_t box[4] = {64, (cuuint32_t)kPxCols, 2, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace unet
}  // namespace ls

using namespace ls::unet;

struct ls_conv_plan {
    CUtensorMap a0, a1, b, y;
    CUtensorMap ys;  // k_conv_upfuse: staged output store (y holds its up weights)
    ConvParamsP p;
    int bn, chunk, grid, mode;
    int mt;    // k_conv_p: 128-pixel sub-tiles per work item
    int full_tiles_y;  // tile rows of the whole layer (row bands restrict p.ty0 / p.tiles_y)
    int kind;  // 0: k_conv_p, 1: k_conv_kx (kx taps stacked along N), 2: k_conv_px2 (pixel pairs)
    int pair;  // k_conv_p on CTA pairs (M = 256 cta_group::2 MMAs, cluster of 2)
    size_t smem;
};

namespace ls {
namespace unet {

// LS_UNET_PDL=0 launches the layers fully serialised (A/B measurements).
static bool pdl_enabled() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_UNET_PDL");
        r = (e && e[0] == '0') ? 0 : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r == 1;
}

// The dynamic shared-memory opt-in of a kernel, once per device: function
// attributes live in each device's context, so a process-wide flag would skip
// the opt-in for the second GPU a plan runs on.
template <typename F>
static int smem_optin(F *fn, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return 0;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSmemBudget + 2048));
    if (e != cudaSuccess) return (int)e;
    done.fetch_or(bit, std::memory_order_acq_rel);
    return 0;
}

// SM count of the current device (plans are sized for the GPU they run on).
static int current_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        return 148;
    return n;
}

template <int BN, int CHUNK, int MODE, int MT>
static int launch_m(const ls_conv_plan *pl, cudaStream_t st) {
    static std::atomic<uint64_t> attr_done{0};  // per-device bits (idempotent races)
    if (int e = smem_optin(k_conv_p<BN, CHUNK, MODE, MT>, attr_done)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl->grid);
    cfg.blockDim = dim3((unsigned)CfgP<BN, CHUNK, MT>::kThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k_conv_p<BN, CHUNK, MODE, MT>, pl->a0, pl->a1, pl->b,
                                   pl->y, pl->p);
}

// CTA-pair launch: clusters of two, at most as many as the device can hold at
// once (queried per device and kernel; the kernel strides its items by the
// cluster count it was launched with).
template <int BN, int CHUNK, int MODE, int MT = 1>
static int launch_pair_m(const ls_conv_plan *pl, cudaStream_t st) {
    auto kern = k_conv_p<BN, CHUNK, MODE, MT, true>;
    static std::atomic<uint64_t> attr_done{0};  // per-device bits (idempotent races)
    if (int e = smem_optin(kern, attr_done)) return e;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return (int)e;
    static std::atomic<int> max_clusters[64];  // per device, 0 = not queried yet
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3((unsigned)CfgP<BN, CHUNK, MT>::kThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    int mc = max_clusters[dev & 63].load(std::memory_order_relaxed);
    if (mc <= 0) {
        cfg.gridDim = dim3((unsigned)pl->grid);
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc <= 0) {
            (void)cudaGetLastError();
            mc = pl->grid / 2;
        }
        max_clusters[dev & 63].store(mc, std::memory_order_relaxed);
    }
    const int clusters = pl->grid / 2 < mc ? pl->grid / 2 : mc;
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.numAttrs = 2;
    return (int)cudaLaunchKernelEx(&cfg, kern, pl->a0, pl->a1, pl->b, pl->y, pl->p);
}

template <int BN, int CHUNK>
static int launch_pair(const ls_conv_plan *pl, cudaStream_t st) {
    if (BN == 128 && pl->mt == 2)
        return pl->mode == kPool ? launch_pair_m<BN, CHUNK, kPool, 2>(pl, st)
                                 : launch_pair_m<BN, CHUNK, kPlain, 2>(pl, st);
    return pl->mode == kPool ? launch_pair_m<BN, CHUNK, kPool>(pl, st)
                             : launch_pair_m<BN, CHUNK, kPlain>(pl, st);
}

template <int CHUNK, int COUT, int MODE>
static int launch_kx_m(const ls_conv_plan *pl, cudaStream_t st) {
    static std::atomic<uint64_t> attr_done{0};  // per-device bits (idempotent races)
    if (int e = smem_optin(k_conv_kx<CHUNK, COUT, MODE>, attr_done)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl->grid);
    cfg.blockDim = dim3((unsigned)CfgKx<CHUNK, COUT>::kThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k_conv_kx<CHUNK, COUT, MODE>, pl->a0, pl->a1, pl->b,
                                   pl->p);
}

template <int CHUNK, int COUT>
static int launch_kx_c(const ls_conv_plan *pl, cudaStream_t st) {
    switch (pl->mode) {
        case kPlain: return launch_kx_m<CHUNK, COUT, kPlain>(pl, st);
        case kPool: return launch_kx_m<CHUNK, COUT, kPool>(pl, st);
        default: return launch_kx_m<CHUNK, COUT, kHead>(pl, st);
    }
}

template <int CHUNK>
static int launch_kx(const ls_conv_plan *pl, cudaStream_t st) {
    return pl->p.cout == 32 ? launch_kx_c<CHUNK, 32>(pl, st) : launch_kx_c<CHUNK, 64>(pl, st);
}

template <int MODE, bool C8, bool KX2 = false, int CO = 32, int CI = 32>
static int launch_px2_m(const ls_conv_plan *pl, cudaStream_t st) {
    static std::atomic<uint64_t> attr_done{0};  // per-device bits (idempotent races)
    if (int e = smem_optin(k_conv_px2<MODE, C8, KX2, CO, CI>, attr_done)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl->grid);
    cfg.blockDim = dim3((unsigned)(64 + 128 * px_groups<KX2 || C8, CO, C8 && !KX2>()));
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k_conv_px2<MODE, C8, KX2, CO, CI>, pl->a0, pl->a1, pl->b,
                                   pl->y, pl->p);
}

static int launch_upfuse(const ls_conv_plan *pl, cudaStream_t st) {
    static std::atomic<uint64_t> attr_done{0};  // per-device bits (idempotent races)
    if (int e = smem_optin(k_conv_upfuse, attr_done)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl->grid);
    cfg.blockDim = dim3((unsigned)(64 + 128 * (kUpGroups + kUpXf)));
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k_conv_upfuse, pl->a0, pl->a1, pl->b, pl->y, pl->ys,
                                   pl->p);
}

static int launch_px2(const ls_conv_plan *pl, cudaStream_t st) {
    if (pl->chunk == 16)  // e0c1: plain only (mt 3: the spill-column form)
        return pl->mt == 3 ? launch_px2_m<kPlain, true, true>(pl, st)
                           : launch_px2_m<kPlain, true>(pl, st);
    if (pl->mt == 1 && pl->bn == 64) {  // neighbour-row pairs, 64 output channels
        if (pl->chunk == 128)
            return pl->mode == kPool ? launch_px2_m<kPool, false, false, 64, 64>(pl, st)
                                     : launch_px2_m<kPlain, false, false, 64, 64>(pl, st);
        return pl->mode == kPool ? launch_px2_m<kPool, false, false, 64, 32>(pl, st)
                                 : launch_px2_m<kPlain, false, false, 64, 32>(pl, st);
    }
    if (pl->mt == 3 && pl->bn == 64) {  // KX2, 64 output channels (chunk 64 / 128: 32 / 64 inputs)
        if (pl->chunk == 128)
            return pl->mode == kPool ? launch_px2_m<kPool, false, true, 64, 64>(pl, st)
                                     : launch_px2_m<kPlain, false, true, 64, 64>(pl, st);
        return pl->mode == kPool ? launch_px2_m<kPool, false, true, 64, 32>(pl, st)
                                 : launch_px2_m<kPlain, false, true, 64, 32>(pl, st);
    }
    if (pl->mt == 3) {  // KX2 variant
        switch (pl->mode) {
            case kPlain: return launch_px2_m<kPlain, false, true>(pl, st);
            case kPool: return launch_px2_m<kPool, false, true>(pl, st);
            default: return launch_px2_m<kHead, false, true>(pl, st);
        }
    }
    switch (pl->mode) {
        case kPlain: return launch_px2_m<kPlain, false>(pl, st);
        case kPool: return launch_px2_m<kPool, false>(pl, st);
        default: return launch_px2_m<kHead, false>(pl, st);
    }
}

static int kx2_setting() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_CONV_KX2");
        r = (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2;
        v.store(r, std::memory_order_relaxed);
    }
    return r;
}

// LS_CONV_PX2 (A/B switch, bit mask, default 3): bit 0 = 32-channel
// single-source layers on k_conv_px2, bit 1 = the 8-channel input layer.
static int px2_mask() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_CONV_PX2");
        r = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 3;
        v.store(r, std::memory_order_relaxed);
    }
    return r;
}

// LS_CONV_KX=0 keeps cout = 32 layers on the generic kernel (A/B measurements).
static bool kx_enabled() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_CONV_KX");
        r = (e && e[0] == '0') ? 0 : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r == 1;
}

template <int BN, int CHUNK, int MT = default_mt(BN)>
static int launch_p(const ls_conv_plan *pl, cudaStream_t st) {
    switch (pl->mode) {
        case kPlain: return launch_m<BN, CHUNK, kPlain, MT>(pl, st);
        case kPool: return launch_m<BN, CHUNK, kPool, MT>(pl, st);
        case kHead: return launch_m<BN, CHUNK, kHead, MT>(pl, st);
        default: return launch_m<BN, CHUNK, kTransposed, MT>(pl, st);
    }
}

// LS_CONV_PAIR: 0 keeps every k_conv_p layer on single-CTA tiles, 1 (default)
// pairs the layers where pair_pays(), 2 pairs every eligible layer (A/B).
static int pair_mode() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_CONV_PAIR");
        r = (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r;
}
static bool pair_enabled() { return pair_mode() != 0; }

static int env_int(const char *name, int dflt);

// smallest column tile on CTA pairs (LS_CONV_PAIR_MINBN, 64 / 128 / 256)
static int pair_min_bn() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        r = env_int("LS_CONV_PAIR_MINBN", 128);
        if (r != 64 && r != 256) r = 128;
        v.store(r, std::memory_order_relaxed);
    }
    return r;
}

static int mt_for(int bn, int h, int w, int batch, int n_tiles_n, bool transposed);

// Pairs only where their coarser work items do not cost more waves: a pair
// item (one 128-pixel sub-tile per SM of the pair) runs ~1.3x faster than a
// single-CTA sub-tile (profiles/README.md, "CTA pairs"), so pair when
// waves(pairs) <= 1.3 x waves(single) x sub-tiles per single item.  The
// 1/16-resolution bottleneck (68 rows: 4.25 pair tiles) stays single.
// Pair tiles: 16 x 16 pixels (the two CTAs' 8-row tiles stacked) or 8 x 32 (side
// by side); the orientation with fewer items wins (the 1/16-resolution
// bottleneck, 68 x 120: 40 stacked vs 36 side-by-side tiles).
static long long pair_items(int h, int w, int batch, int n_tiles_n, bool side) {
    const long long tx = side ? (w + 2 * kTW - 1) / (2 * kTW) : (w + kTW - 1) / kTW;
    const long long ty = side ? (h + kTH - 1) / kTH : (h + 2 * kTH - 1) / (2 * kTH);
    return tx * ty * batch * n_tiles_n;
}
static bool pair_side(int h, int w, int batch, int n_tiles_n) {
    const int e = env_int("LS_CONV_PAIR_SIDE", 2);  // A/B: 0 stacked, 1 side by side
    if (e != 2) return e == 1;
    return pair_items(h, w, batch, n_tiles_n, true) < pair_items(h, w, batch, n_tiles_n, false);
}

static bool pair_pays(int bn, int h, int w, int batch, int n_tiles_n) {
    if (pair_mode() == 2) return true;
    const int n_sm = current_sm_count();
    const long long tx = (w + kTW - 1) / kTW;
    const long long items_p = pair_items(h, w, batch, n_tiles_n, pair_side(h, w, batch, n_tiles_n));
    const long long waves_p = (items_p + n_sm / 2 - 1) / (n_sm / 2);
    const int mt = mt_for(bn, h, w, batch, n_tiles_n, false);
    const long long items_s = tx * ((h + kTH * mt - 1) / (kTH * mt)) * batch * n_tiles_n;
    const long long waves_s = (items_s + n_sm - 1) / n_sm;
    return 10 * waves_p <= 13 * waves_s * mt;
}

// LS_CONV_MT2=0 keeps 256-column tiles at one sub-tile per item (A/B).
static bool mt2_enabled() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_CONV_MT2");
        r = (e && e[0] == '0') ? 0 : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r == 1;
}

// A/B knobs of the tile shape (defaults = the product shapes):
//   LS_CONV_N256=128   256-output-channel layers on 128-column tiles
//   LS_CONV_MT128=2    128-column tiles with two 128-pixel sub-tiles per item
static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

static int mt_for(int bn, int h, int w, int batch, int n_tiles_n, bool transposed) {
    if (bn == 128 && !transposed && env_int("LS_CONV_MT128", 1) == 2) return 2;
    const int mt = default_mt(bn);
    if (bn == 256 && mt == 1 && !transposed && mt2_enabled()) {
        const int items2 = ((w + kTW - 1) / kTW) * ((h + 2 * kTH - 1) / (2 * kTH)) * batch * n_tiles_n;
        const int n_sm = current_sm_count();
        if (items2 * 5 >= n_sm * 4) return 2;
    }
    return mt;
}

}  // namespace unet
}  // namespace ls

static bool chunk_ok(int c) { return c == 16 || c == 32 || (c > 0 && c % 64 == 0); }

// Plan of a 32 -> 32 (or [32, 32] -> 32) 3x3 layer on k_conv_px2 (null when
// it does not apply: odd width).
static ls_conv_plan *plan_px2(bool kx2, const uint16_t *d_x0, int c0, const uint16_t *d_x1, int c1,
                              int cout, int batch,
                              int h, int w, const uint16_t *d_w, const float *d_scale,
                              const float *d_shift, int act, float alpha, uint16_t *d_y,
                              float *d_y_f32, uint16_t *d_pool, const float *d_head_w,
                              const float *d_head_b, int head_c, float *d_head_out) {
    using namespace ls::unet;
    if (w % 2) return nullptr;
    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan();
    if (!pl) return nullptr;
    ConvParamsP &p = pl->p;
    p = ConvParamsP{};
    p.batch = batch;
    p.h = h;
    p.w = w;
    const bool c8 = c0 == 8;
    // 64-channel forms (KX2 or neighbour-row): cout 64, inputs of 32 or 64
    // channels (one source)
    if (cout != 32 && !(cout == 64 && c1 == 0 && (c0 == 32 || c0 == 64))) {
        delete pl;
        return nullptr;
    }
    const bool ci64 = c0 == 64;
    p.c0 = c8 ? 16 : c0;
    p.c1 = c1;
    p.ctot = p.c0 + c1;
    p.wts = d_w;
    if (cudaMemcpy(p.pc_scale, d_scale, cout * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(p.pc_shift, d_shift, cout * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
        (d_head_w && cudaMemcpy(p.pc_head, d_head_w, (size_t)head_c * 32 * sizeof(float),
                                cudaMemcpyDeviceToHost) != cudaSuccess)) {
        delete pl;
        return nullptr;
    }
    p.kxs = 3;
    p.kxps = 1;
    p.pad = 1;
    p.n_total = cout;
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
    p.tiles_x = (w / 2 + kPxCols - 1) / kPxCols;
    p.tiles_y = (h + kTH - 1) / kTH;
    p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
    p.n_tiles_n = 1;
    p.n_items = p.n_tiles_m;
    p.nq0 = 1;
    p.nq = c1 > 0 ? 2 : 1;
    const uint32_t arow = c8 ? 32u : CfgPx::kRow;
    p.a_tx = (uint32_t)(kTW * (kTH + 2)) * arow;
    p.a_bytes = (p.a_tx + 1023u) & ~1023u;
    p.b_blk = CfgPx::kBTile;
    p.resident = 1;
    // KX2 B tiles: per (source, ky, K16 step) 3 x cout rows x 32 B; neighbour-row
    // tiles: per (source, ky, element, K16 step) 2 x cout rows x 32 B
    const size_t res_bytes = c8 ? (size_t)3 * 4096
                                : (kx2 ? (size_t)p.nq * 3 * (p.c0 / 16) * 3 * cout * 32
                                       : (size_t)p.nq * 3 * 2 * (p.c0 / 16) * 2 * cout * 32);
    const size_t const_bytes =
        ((size_t)(2 * cout + (d_head_w ? head_c * 32 : 0)) * 4 + 1023) & ~size_t(1023);
    // 32-channel bf16 outputs leave through per-warp shared-memory staging
    // buffers (4 KB: two tile rows x 14 pairs x 128 B) and TMA stores
    const bool c8kx2 = c8 && env_int("LS_CONV_C8KX2", 0) == 1;
    const int groups = c8 ? (c8kx2 ? LS_KX2_GROUPS : LS_C8_GROUPS)
                          : kx2 ? (cout == 64 ? LS_KX2_64_GROUPS : LS_KX2_GROUPS)
                                : CfgPx::kEpiGroups;
    // (LS_PX_STAGE: 2 buffers per warp, so a store's read of one overlaps the
    // next item's writes into the other -- one when that leaves < 4 ring stages;
    // 1: one buffer; 0: lane stores)
    int bufs = cout == 32 && d_y && !d_y_f32 ? env_int("LS_PX_STAGE", 2) : 0;
    if (bufs < 0 || bufs > 2) bufs = 2;
    const uint32_t stage_bytes = (ci64 ? 2u : 1u) * p.a_bytes;  // 64-ch inputs: two element boxes
    size_t stage_total;
    int stages;
    for (;;) {
        stage_total = (size_t)bufs * groups * 4 * 4096;
        const size_t fixed =
            CfgPx::kRingPad + res_bytes + const_bytes + stage_total + (stage_total ? 1024 : 0) + 512;
        stages = kSmemBudget > fixed ? (int)((kSmemBudget - fixed) / stage_bytes) : 0;
        if (bufs == 2 && stages < 4) {
            bufs = 1;
            continue;
        }
        break;
    }
    p.stage_store = bufs;
    if (stages < 3) {
        delete pl;
        return nullptr;
    }
    if (stages > 8) stages = 8;
    p.stages = stages;
    p.stage_bytes = stage_bytes;
    p.off_b = (uint32_t)(CfgPx::kRingPad + stages * p.stage_bytes);
    p.off_const = (uint32_t)(p.off_b + res_bytes);
    p.off_pool = (uint32_t)(p.off_const + const_bytes);
    p.off_stage = (p.off_pool + 1023u) & ~1023u;
    p.off_bar = (uint32_t)(p.off_stage + stage_total);
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = cout;
    pl->chunk = c8 ? 16 : 2 * c0;  // pair-row channels (128: two 64-channel element boxes)
    pl->kind = 2;
    // 3 marks the KX2 (spill-column) variant; the 8-channel layer stays on the
    // neighbour-row form unless LS_CONV_C8KX2=1 (one N = 128 MMA per ky instead of
    // three, but the spill-column epilogue: e0c1 47 -> 52 us, measured slower)
    pl->mt = (kx2 && !c8) || c8kx2 ? 3 : 1;
    pl->mode = d_head_w ? kHead : (d_pool ? kPool : kPlain);
    const int n_sm = current_sm_count();
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    pl->full_tiles_y = p.tiles_y;
    // the NHWC tensors read as (W/2) pair pixels of 2*c channels (64-channel
    // inputs: one box per element)
    const int pc = c8 ? 16 : 64;
    bool ok;
    if (ci64) {
        ok = encode_act_pairsplit(&pl->a0, d_x0, w, h, batch, kTH + 2);
        pl->a1 = pl->a0;
    } else {
        ok = encode_act(&pl->a0, d_x0, pc, w / 2, h, batch, pc, kTH + 2);
        ok = ok && encode_act(&pl->a1, c1 > 0 ? d_x1 : d_x0, pc, w / 2, h, batch, pc, kTH + 2);
    }
    ok = ok && encode_wts(&pl->b, d_w, p.ctot, cout, 9, 16, cout, 1);
    ok = ok && (!p.stage_store || encode_pair_store(&pl->y, d_y, w, h, batch));
    if (!ok) {
        delete pl;
        return nullptr;
    }
    return pl;
}

// Plan of a cout = 32 / 64, 3x3 layer on k_conv_kx (null when it does not
// fit).  c0 is the K-chunk channel count of source 0 (8 -> 16), c0_tensor
// its tensor's.
static ls_conv_plan *plan_kx(const uint16_t *d_x0, int c0_tensor, int c0, const uint16_t *d_x1,
                             int c1, int cout, int batch, int h, int w, const uint16_t *d_w,
                             const float *d_scale, const float *d_shift, int act, float alpha,
                             uint16_t *d_y, float *d_y_f32, uint16_t *d_pool,
                             const float *d_head_w, const float *d_head_b, int head_c,
                             float *d_head_out) {
    using namespace ls::unet;
    int chunk = 64;
    while (chunk > 16 && ((c0 % chunk) || (c1 % chunk))) chunk >>= 1;
    if ((c0 % chunk) || (c1 % chunk)) return nullptr;
    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan();
    if (!pl) return nullptr;
    ConvParamsP &p = pl->p;
    p = ConvParamsP{};
    p.batch = batch;
    p.h = h;
    p.w = w;
    p.c0 = c0;
    p.c1 = c1;
    p.ctot = c0 + c1;
    p.kxs = 3;
    p.kxps = 1;
    p.pad = 1;
    p.n_total = cout;
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
    p.tiles_x = (w + kKxCols - 1) / kKxCols;
    p.tiles_y = (h + kTH - 1) / kTH;
    p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
    p.n_tiles_n = 1;
    p.n_items = p.n_tiles_m;
    p.nq0 = c0 / chunk;
    p.nq = (c0 + c1) / chunk;
    const uint32_t row = (uint32_t)chunk * 2;
    p.a_tx = (uint32_t)(kTW * (kTH + 2)) * row;
    p.a_bytes = (p.a_tx + 1023u) & ~1023u;
    p.b_blk = (uint32_t)cout * row;
    p.resident = 1;
    const size_t res_bytes = (size_t)9 * p.nq * p.b_blk;
    const size_t const_bytes =
        ((size_t)(2 * cout + (d_head_w ? head_c * cout : 0)) * 4 + 1023) & ~size_t(1023);
    const size_t fixed = res_bytes + const_bytes + 512;
    int stages = kSmemBudget > fixed ? (int)((kSmemBudget - fixed) / p.a_bytes) : 0;
    if (stages < 3) {
        delete pl;
        return nullptr;
    }
    if (stages > 8) stages = 8;
    p.stages = stages;
    p.stage_bytes = p.a_bytes;
    p.off_b = (uint32_t)(stages * p.stage_bytes);
    p.off_const = (uint32_t)(p.off_b + res_bytes);
    p.off_pool = (uint32_t)(p.off_const + const_bytes);
    p.off_bar = p.off_pool;
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = cout;
    pl->chunk = chunk;
    pl->kind = 1;
    pl->mode = d_head_w ? kHead : (d_pool ? kPool : kPlain);
    const int n_sm = current_sm_count();
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    pl->full_tiles_y = p.tiles_y;
    bool ok = encode_act(&pl->a0, d_x0, c0_tensor, w, h, batch, chunk, kTH + 2);
    ok = ok && encode_act(&pl->a1, c1 > 0 ? d_x1 : d_x0, c1 > 0 ? c1 : c0_tensor, w, h, batch,
                          chunk, kTH + 2);
    ok = ok && encode_wts(&pl->b, d_w, p.ctot, cout, 9, chunk, cout, 1);
    if (!ok) {
        delete pl;
        return nullptr;
    }
    return pl;
}

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
    // c0 = 8 (single source): the tensor has 8 channels per pixel and is read
    // as a 16-channel K chunk whose upper half the TMA zero-fills (box wider
    // than the tensor's channel extent) -- the network input's 5 live
    // channels at half the bytes of a 16-channel layout
    const int c0_tensor = c0;
    if (c0 == 8 && c1 == 0) c0 = 16;
    if (!d_x0 || !d_w || !d_scale || !d_shift || batch < 1 || h < 1 || w < 1 || !chunk_ok(c0))
        return fail(LS_EINVAL);
    if (c1 < 0 || (c1 > 0 && (!d_x1 || !chunk_ok(c1)))) return fail(LS_EINVAL);
    if (cout < 16 || cout % 16 || (ksize != 1 && ksize != 3)) return fail(LS_EINVAL);
    // the fused epilogue evaluates leaky ReLU as max(v, alpha * v)
    if (act == LS_ACT_LEAKY && !(alpha >= 0.0f && alpha <= 1.0f)) return fail(LS_EINVAL);
    if (transposed && (ksize != 1 || c1 != 0 || d_pool || d_head_w)) return fail(LS_EINVAL);
    if (!transposed && ksize != 3) return fail(LS_EINVAL);  // 1x1 convs are fused heads
    if (d_pool && (h % 2 || w % 2)) return fail(LS_EINVAL);
    if (d_head_w && (head_c < 1 || head_c > 4 || !d_head_b || !d_head_out)) return fail(LS_EINVAL);
    const int n_total = transposed ? 4 * cout : cout;
    if (n_total > 4096) return fail(LS_EINVAL);
    // cout = 64 items hold 192 TMEM columns (2 buffers): worth it only when the
    // K loop is long enough to cover the buffer round trip (measured: K = 128
    // 94 -> 66 us, K = 32 / 64 slower)
    // pixel-pair kernels (k_conv_px2): the KX2 variant (spill columns) for the
    // 32-channel layers (measured U-Net 0.893 ms with neighbour-row MMAs for the
    // single-source layers and k_conv_kx for d0c1, 0.879 with KX2 on d0c1 only,
    // 0.873 with KX2 everywhere; LS_CONV_KX2=1: d0c1 only, 0: never), the
    // neighbour-row form for the 8-channel input layer
    const int kx2_mode = kx2_setting();
    const bool kx2 = cout == 32 && c0_tensor == 32 && (c1 == 0 || c1 == 32) &&
                     (kx2_mode == 2 || (kx2_mode == 1 && c1 == 32));
    // 64-channel single-source layers (enc1 conv1 / conv2, dec1 conv2) on the
    // KX2 pixel-pair form (LS_CONV_KX2_64=0: k_conv_p)
    const bool kx2_64 = cout == 64 && c1 == 0 && (c0_tensor == 32 || c0_tensor == 64) &&
                        !d_head_w && env_int("LS_CONV_KX2_64", 1) != 0;
    const bool px2_fit = kx2 || kx2_64 || (cout == 32 && c1 == 0 &&
                         ((c0_tensor == 32 && (px2_mask() & 1)) ||
                          (c0_tensor == 8 && !d_pool && !d_head_w && (px2_mask() & 2))));
    if (!transposed && px2_fit) {
        // 64-channel layers: the neighbour-row form (4 TMEM buffers of 128 columns)
        // for 32-channel inputs, whose short K loop leaves the 2-buffer KX2 form
        // waiting on its accumulator round trip (e1c1 35.8 -> 30.5 us), KX2 for
        // 64-channel inputs (e1c2 43.4 vs 49.7, d1c2 41.0 vs 42.5 us).
        // LS_CONV_PX64: 0 = KX2 always, 1 = neighbour-row always, 2 = by input
        const int px64 = env_int("LS_CONV_PX64", 2);
        const bool nbr64 = kx2_64 && (px64 == 1 || (px64 == 2 && c0_tensor == 32));
        ls_conv_plan *pp = plan_px2(kx2 || (kx2_64 && !nbr64), d_x0, c0_tensor, d_x1, c1, cout, batch, h, w,
                                    d_w, d_scale, d_shift, act,
                                    alpha, d_y, d_y_f32, d_pool, d_head_w, d_head_b, head_c,
                                    d_head_out);
        if (pp) {
            if (status) *status = 0;
            return pp;
        }
    }
    const bool kx_fit = cout == 32 || (cout == 64 && c0 + c1 >= 128 && !d_head_w);
    if (!transposed && kx_fit && kx_enabled()) {
        ls_conv_plan *pk = plan_kx(d_x0, c0_tensor, c0, d_x1, c1, cout, batch, h, w, d_w, d_scale,
                                   d_shift,
                                   act, alpha, d_y, d_y_f32, d_pool, d_head_w, d_head_b, head_c,
                                   d_head_out);
        if (pk) {
            if (status) *status = 0;
            return pk;
        }  // no fit: fall through to the generic kernel
    }
    int bn = n_total >= 256 ? 256 : (n_total >= 128 ? 128 : (n_total >= 64 ? 64 : 32));
    if (n_total % bn) bn = 32;
    // 256-channel layers on 128-column tiles: with CTA pairs (M = 256) the twice
    // as many items balance better over the SMs (measured 0.810 -> 0.804 ms;
    // LS_CONV_N256=256 keeps 256-column tiles)
    if (bn == 256 && n_total == 256 && !transposed && !d_head_w &&
        env_int("LS_CONV_N256", pair_enabled() ? 128 : 256) == 128)
        bn = 128;
    {
        // small grids (the 1/16-resolution bottleneck): 128-column tiles when
        // 256-column ones leave SMs idle (LS_CONV_SMALLN=0 keeps 256)
        const int n_sm = current_sm_count();
        const long long m_tiles = (long long)((w + kTW - 1) / kTW) * ((h + kTH - 1) / kTH) * batch;
        const char *e = getenv("LS_CONV_SMALLN");
        if (bn == 256 && !transposed && !d_head_w && !(e && e[0] == '0') &&
            m_tiles * (n_total / 256) < n_sm)
            bn = 128;
    }
    // transposed convs are epilogue-bound (K is small, 4x cout outputs per
    // input pixel): 128-column tiles leave room for 3 epilogue warpgroups
    // (LS_CONV_UPBN=256: 256-column tiles, A/B)
    if (transposed && bn > 128 && env_int("LS_CONV_UPBN", 128) != 256) bn = 128;
    if (d_head_w && n_total > bn) return fail(LS_EINVAL);  // the head needs every channel
    int chunk = bn >= 256 ? 32 : 64;
    while (chunk > 16 && ((c0 % chunk) || (c1 % chunk))) chunk >>= 1;

    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan();
    if (!pl) return fail(LS_EINVAL);
    pl->kind = 0;
    ConvParamsP &p = pl->p;
    p.batch = batch;
    p.h = h;
    p.w = w;
    p.c0 = c0;
    p.c1 = c1;
    p.ctot = c0 + c1;
    p.kxs = ksize == 3 ? 3 : 1;
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
    const int kys = p.kxs;
    const size_t const_bytes = ((size_t)(2 * n_total + (d_head_w ? head_c * cout : 0)) * 4 + 1023) &
                               ~size_t(1023);
    size_t res_bytes = 0;
    int stages = 0;
    // staged TMA stores for 32-channel transposed convs (LS_CONV_UPSTORE=0: off)
    const char *ue = getenv("LS_CONV_UPSTORE");
    // (cout 64: the staged box spans the image boundary when rows are ragged, so
    // batches need h % 8 == 0)
    const bool want_stage = transposed && d_y && !d_y_f32 && !(ue && ue[0] == '0') &&
                            (cout == 32 || (cout == 64 && (batch == 1 || h % kTH == 0)));
    // Fit >= 3 pipeline stages: first try whole-chunk stages (all kx boxes in
    // one stage), then one kx per stage, then a narrower K chunk, then a
    // narrower column tile.
    int mt = 1;
    // CTA pairs for the plain / pooling layers with >= 128-column tiles
    // (LS_CONV_PAIR=0: single-CTA tiles everywhere)
    bool pair = !transposed && !d_head_w && bn >= pair_min_bn() && pair_enabled() &&
                pair_pays(bn, h, w, batch, (n_total + bn - 1) / bn);
    for (;;) {
        if (bn < pair_min_bn() || chunk < 16) pair = false;
        mt = pair ? (bn == 128 ? env_int("LS_CONV_PAIR_MT", 1) == 2 ? 2 : 1 : 1)
                  : mt_for(bn, h, w, batch, (n_total + bn - 1) / bn, transposed != 0);
        // transposed convs without staged stores (cout >= 128): two 128-pixel
        // sub-tiles per item share each streamed weight block (LS_CONV_UPMT)
        if (transposed && !want_stage && bn == 128 && env_int("LS_CONV_UPMT", 1) == 2) mt = 2;
        const int box_h = kTH * mt + 2 * p.pad;
        p.pair_h = pair && pair_side(h, w, batch, (n_total + bn - 1) / bn) ? 1 : 0;
        const int tile_h = kTH * mt * (pair && !p.pair_h ? 2 : 1);
        const int tile_w = kTW * (p.pair_h ? 2 : 1);
        const uint32_t row = (uint32_t)chunk * 2;
        p.tiles_x = (w + tile_w - 1) / tile_w;
        p.tiles_y = (h + tile_h - 1) / tile_h;
        p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
        p.n_tiles_n = (n_total + bn - 1) / bn;
        p.n_items = p.n_tiles_m * p.n_tiles_n;
        p.nq0 = c0 / chunk;
        p.nq = (c0 + c1) / chunk;
        p.a_tx = (uint32_t)(kTW * box_h) * row;
        p.a_bytes = (p.a_tx + 1023u) & ~1023u;
        p.b_blk = (uint32_t)(kys * (pair ? bn / 2 : bn)) * row;
        const size_t nk = (size_t)p.kxs * p.nq;
        p.resident = (p.n_tiles_n == 1 && nk * p.b_blk <= kResidentMax) ? 1 : 0;
        res_bytes = p.resident ? nk * p.b_blk : 0;
        const bool stage_now = want_stage && bn == 128 && mt == 1;
        const size_t fixed = res_bytes + const_bytes + 512 + (stage_now ? 3 * 32768 + 1024 : 0);
        bool fit = false;
        for (int kxps = p.kxs; kxps >= 1 && !fit; kxps = kxps == 1 ? 0 : 1) {
            const size_t stage_bytes = (size_t)kxps * (p.a_bytes + (p.resident ? 0 : p.b_blk));
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
    p.off_pool = (uint32_t)(p.off_const + const_bytes);
    p.stage_store = want_stage && bn == 128 && mt == 1 ? 1 : 0;
    if (p.stage_store) {
        p.off_stage = (p.off_pool + 1023u) & ~1023u;
        p.off_pool = p.off_stage + 3 * 32768;
    }
    p.off_bar = p.off_pool;
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = bn;
    pl->chunk = chunk;
    pl->pair = pair ? 1 : 0;
    pl->mode = transposed ? kTransposed : (d_head_w ? kHead : (d_pool ? kPool : kPlain));
    if (p.stage_store && !(cout == 64 ? encode_up_store64(&pl->y, d_y, w, h, batch)
                                      : encode_up_store(&pl->y, d_y, w, h, batch))) {
        delete pl;
        return fail(LS_EINVAL);
    }
    const int n_sm = current_sm_count();
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    if (pair) pl->grid = 2 * (p.n_items < n_sm / 2 ? p.n_items : n_sm / 2);
    pl->full_tiles_y = p.tiles_y;
    const int box_h = kTH * mt + 2 * p.pad;
    pl->mt = mt;
    bool ok = encode_act(&pl->a0, d_x0, c0_tensor, w, h, batch, chunk, box_h);
    ok = ok && encode_act(&pl->a1, c1 > 0 ? d_x1 : d_x0, c1 > 0 ? c1 : c0_tensor, w, h, batch,
                          chunk, box_h);
    ok = ok && encode_wts(&pl->b, d_w, p.ctot, n_total, p.kxs * kys, chunk, pair ? bn / 2 : bn, kys);
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
    if (pl->kind == 2) return launch_px2(pl, st);
    if (pl->kind == 3) return launch_upfuse(pl, st);
    if (pl->pair) {
        if (pl->bn == 128 && pl->chunk == 64) return launch_pair<128, 64>(pl, st);
        if (pl->bn == 128 && pl->chunk == 32) return launch_pair<128, 32>(pl, st);
        if (pl->bn == 256 && pl->chunk == 32) return launch_pair<256, 32>(pl, st);
        if (pl->bn == 256 && pl->chunk == 16) return launch_pair<256, 16>(pl, st);
        if (pl->bn == 64 && pl->chunk == 64) return launch_pair<64, 64>(pl, st);
        if (pl->bn == 64 && pl->chunk == 32) return launch_pair<64, 32>(pl, st);
        return LS_EINVAL;
    }
    if (pl->kind == 1) {
        if (pl->chunk == 16) return launch_kx<16>(pl, st);
        if (pl->chunk == 32) return launch_kx<32>(pl, st);
        return launch_kx<64>(pl, st);
    }
#define LS_CASE(B, K) \
    if (pl->bn == B && pl->chunk == K && pl->mt == default_mt(B)) return launch_p<B, K>(pl, st);
    LS_CASE(32, 16) LS_CASE(32, 32) LS_CASE(32, 64)
    LS_CASE(64, 16) LS_CASE(64, 32) LS_CASE(64, 64)
    LS_CASE(128, 16) LS_CASE(128, 32) LS_CASE(128, 64)
    LS_CASE(256, 16) LS_CASE(256, 32)
#undef LS_CASE
    if (pl->bn == 256 && pl->chunk == 32 && pl->mt == 2) return launch_p<256, 32, 2>(pl, st);
    if (pl->bn == 128 && pl->chunk == 64 && pl->mt == 2) return launch_p<128, 64, 2>(pl, st);
    if (pl->bn == 128 && pl->chunk == 32 && pl->mt == 2) return launch_p<128, 32, 2>(pl, st);
    if (pl->bn == 256 && pl->chunk == 16 && pl->mt == 2) return launch_p<256, 16, 2>(pl, st);
    return LS_EINVAL;
}

void ls_conv_plan_destroy(ls_conv_plan *pl) { delete pl; }

ls_conv_plan *ls_conv_plan_create_upfused(const uint16_t *d_x, const uint16_t *d_up_w,
                                          const float *d_up_shift, const uint16_t *d_skip,
                                          int32_t batch, int32_t h, int32_t w, const uint16_t *d_w,
                                          const float *d_scale, const float *d_shift, int32_t act,
                                          float alpha, uint16_t *d_y, int32_t *status) {
    using namespace ls::unet;
    auto fail = [&](int32_t e) -> ls_conv_plan * {
        if (status) *status = e;
        return nullptr;
    };
    if (!d_x || !d_up_w || !d_up_shift || !d_skip || !d_w || !d_scale || !d_shift || !d_y ||
        batch < 1 || h < 2 || w < 2 || (h % 2) || (w % 2) || (act != LS_ACT_NONE && act != LS_ACT_RELU &&
                                                        act != LS_ACT_LEAKY))
        return fail(LS_EINVAL);
    ls_conv_plan *pl = new (std::nothrow) ls_conv_plan();
    if (!pl) return fail(LS_EINVAL);
    ConvParamsP &p = pl->p;
    p = ConvParamsP{};
    p.batch = batch;
    p.h = h;
    p.w = w;
    p.c0 = 32;
    p.c1 = 32;
    p.ctot = 64;
    p.nq0 = 1;
    p.nq = 2;
    p.kxs = 3;
    p.kxps = 1;
    p.pad = 1;
    p.n_total = 32;
    p.cout = 32;
    p.act = act;
    p.alpha = alpha;
    p.scale = d_scale;
    p.shift = d_shift;
    p.y = reinterpret_cast<__nv_bfloat16 *>(d_y);
    if (cudaMemcpy(p.pc_scale, d_scale, 32 * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(p.pc_shift, d_shift, 32 * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(p.pc_upb, d_up_shift, 32 * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) {
        delete pl;
        return fail(LS_EINVAL);
    }
    p.tiles_x = (w / 2 + kPxCols - 1) / kPxCols;
    p.tiles_y = (h + kTH - 1) / kTH;
    p.n_tiles_m = p.tiles_x * p.tiles_y * batch;
    p.n_tiles_n = 1;
    p.n_items = p.n_tiles_m;
    p.a_tx = kUpBox;  // the skip box; the dec1 box is 16 KB
    p.a_bytes = kUpBox;
    p.stage_bytes = kUpBox;
    p.resident = 1;
    const size_t res_bytes = 12 * 3072 + 16384;  // KX2 tiles of both sources + up weights
    const size_t boxes = 2 * (size_t)kUpBox;     // the transform's two source-0 boxes
    // staged output stores (4 KB per epilogue warp, LS_UPF_STAGE=1) when the ring
    // keeps >= 4 stages
    const size_t ystage = (size_t)kUpGroups * 4 * 4096;
    p.stage_store = env_int("LS_UPF_STAGE", 1) == 1 ? 1 : 0;
    int stages = 0;
    for (;;) {
        const size_t fixed =
            CfgPx::kRingPad + boxes + res_bytes + (p.stage_store ? ystage + 1024 : 0) + 512;
        stages = kSmemBudget > fixed ? (int)((kSmemBudget - fixed) / p.stage_bytes) : 0;
        stages &= ~1;  // two ring stages per item
        if (p.stage_store && stages < 4) {
            p.stage_store = 0;
            continue;
        }
        break;
    }
    if (stages < 4) {
        delete pl;
        return fail(LS_EINVAL);
    }
    if (stages > 8) stages = 8;
    p.stages = stages;
    p.off_stage = (uint32_t)(CfgPx::kRingPad + stages * p.stage_bytes);
    p.off_b = (uint32_t)(p.off_stage + boxes);
    p.off_const = (uint32_t)(p.off_b + res_bytes);
    p.off_pool = p.stage_store ? (p.off_const + 1023u) & ~1023u : p.off_const;  // output staging
    p.off_bar = p.off_pool + (p.stage_store ? (uint32_t)ystage : 0u);
    pl->smem = 1024 + p.off_bar + 512;
    pl->bn = 32;
    pl->chunk = 64;
    pl->kind = 3;
    pl->mt = 1;
    pl->mode = kPlain;
    const int n_sm = current_sm_count();
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    pl->full_tiles_y = p.tiles_y;
    // dec1 output [n][h/2][w/2][64] as boxes {64, 16, 8}; skip as pair pixels
    bool ok = encode_act(&pl->a0, d_x, 64, w / 2, h / 2, batch, 64, 8);
    ok = ok && encode_act(&pl->a1, d_skip, 64, w / 2, h, batch, 64, kTH + 2);
    ok = ok && encode_wts(&pl->b, d_w, 64, 32, 9, 16, 32, 1);
    ok = ok && encode_wts(&pl->y, d_up_w, 64, 128, 1, 64, 128, 1);
    ok = ok && (!p.stage_store || encode_pair_store(&pl->ys, d_y, w, h, batch));
    if (!ok) {
        delete pl;
        return fail(LS_EINVAL);
    }
    if (status) *status = 0;
    return pl;
}

int ls_conv_plan_set_reverse(ls_conv_plan *pl, int32_t reverse) {
    if (!pl) return LS_EINVAL;
    pl->p.reverse = reverse ? 1 : 0;
    return 0;
}

int ls_conv_plan_set_rows(ls_conv_plan *pl, int32_t row_begin, int32_t row_end) {
    if (!pl) return LS_EINVAL;
    const int th = pl->kind == 0 ? kTH * pl->mt * (pl->pair && !pl->p.pair_h ? 2 : 1) : kTH;
    const int h = pl->p.h;
    if (row_begin < 0 || row_end > h || row_begin >= row_end || row_begin % th) return LS_EINVAL;
    const int t0 = row_begin / th, t1 = (row_end + th - 1) / th;
    if (t1 > pl->full_tiles_y) return LS_EINVAL;
    ConvParamsP &p = pl->p;
    p.ty0 = t0;
    p.tiles_y = t1 - t0;
    p.n_tiles_m = p.tiles_x * p.tiles_y * p.batch;
    p.n_items = p.n_tiles_m * p.n_tiles_n;
    const int n_sm = current_sm_count();
    pl->grid = p.n_items < n_sm ? p.n_items : n_sm;
    return 0;
}

int32_t ls_conv_plan_tile_rows(const ls_conv_plan *pl) {
    if (!pl) return LS_EINVAL;
    return pl->kind == 0 ? kTH * pl->mt * (pl->pair && !pl->p.pair_h ? 2 : 1) : kTH;
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
