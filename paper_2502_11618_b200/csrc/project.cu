// Projection: the two-pass deterministic soft z-buffer (render.py:84-161).
//
// Pass 1 folds the per-pixel minimum camera depth with a 64-bit atomicMin on
// the f64 bit pattern of zc (zc >= z_near > 0, and positive IEEE doubles order
// like unsigned integers), preceded by a plain L2 read so only improving points
// pay for an atomic.  Pass 2 recomputes pixel and depth (cheaper than the
// reference's 16 B/point pix_cache/z_cache round trip) and integer-accumulates
// colours of every point within the soft tolerance.  Both reductions are
// order-free, so the result is bit-identical to the reference for any
// schedule (reference render.py:1-12).
//
// Fast path layout: warp tiles of LS_TILE_POINTS = 128 cell-major points; each
// lane owns 4 consecutive points = 48 contiguous bytes (3 x LDG.128) of xyz and
// 12 bytes (3 x LDG.32) of rgb.  Per-tile occupied-cell spans (built once per
// scan) let a warp skip a fully culled tile without touching its points.
#include <atomic>
#include <mutex>
#include <cuda_fp16.h>
#include "ls_common.cuh"
#include "umma.cuh"

#include <stdlib.h>

#include <type_traits>

namespace ls {

const void *cull_kernel();
int cull_planes_arg();

// ---------------------------------------------------------------------------
// (i) twins with the reference's range/cache interface
// ---------------------------------------------------------------------------

// Exclusive prefix of range lengths (n_ranges is small; one CTA, serial carry).
__global__ void k_range_prefix(const int64_t *__restrict__ starts, const int64_t *__restrict__ ends,
                               int64_t nr, int64_t *__restrict__ prefix) {
    __shared__ int64_t carry;
    __shared__ int64_t warp_tot[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nr; base += blockDim.x) {
        int64_t r = base + threadIdx.x;
        int64_t len = r < nr ? ends[r] - starts[r] : 0;
        // block inclusive scan
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int64_t v = len;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) warp_tot[wid] = v;
        __syncthreads();
        if (wid == 0) {
            int64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int64_t u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        int64_t incl = v + (wid > 0 ? warp_tot[wid - 1] : 0) + carry;
        if (r < nr) prefix[r] = incl - len;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) prefix[nr] = carry;
}

__device__ __forceinline__ int64_t find_range(const int64_t *__restrict__ prefix, int64_t nr,
                                              int64_t k) {
    // largest r with prefix[r] <= k (ranges may be empty)
    int64_t lo = 0, hi = nr - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_twin_pass1(const float *__restrict__ pos, const int64_t *__restrict__ starts,
                             const int64_t *__restrict__ prefix, int64_t nr, ProjCam c,
                             unsigned long long *__restrict__ minz, int64_t *__restrict__ pix_cache,
                             double *__restrict__ z_cache) {
    const int64_t n = prefix[nr];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = find_range(prefix, nr, k);
        int64_t i = starts[r] + (k - prefix[r]);
        double zc;
        int64_t pix = project_point(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], c, zc);
        z_cache[k] = zc;
        pix_cache[k] = pix;
        if (pix >= 0) {
            // caller minz is f64; comparisons on bits are valid for zc > 0 and
            // any non-negative minz (the only values a z_near > 0 pass produces)
            unsigned long long key = (unsigned long long)__double_as_longlong(zc);
            if (key < __ldcg(minz + pix)) atomicMin(minz + pix, key);
        }
    }
}

__global__ void k_twin_pass2(const uint8_t *__restrict__ col, const int64_t *__restrict__ starts,
                             const int64_t *__restrict__ prefix, int64_t nr,
                             const int64_t *__restrict__ pix_cache,
                             const double *__restrict__ z_cache, double ope,
                             const double *__restrict__ minz,
                             unsigned long long *__restrict__ accum) {
    const int64_t n = prefix[nr];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t pix = pix_cache[k];
        if (pix < 0) continue;
        if (!(z_cache[k] <= dmul(minz[pix], ope))) continue;
        int64_t r = find_range(prefix, nr, k);
        int64_t i = starts[r] + (k - prefix[r]);
        unsigned long long *a = accum + 4 * pix;
        atomicAdd(a + 0, (unsigned long long)col[3 * i + 0]);
        atomicAdd(a + 1, (unsigned long long)col[3 * i + 1]);
        atomicAdd(a + 2, (unsigned long long)col[3 * i + 2]);
        atomicAdd(a + 3, 1ull);
    }
}

__global__ void k_assemble_exact(const double *__restrict__ minz,
                                 const unsigned long long *__restrict__ accum, int64_t npix,
                                 float *__restrict__ rgb, float *__restrict__ depth,
                                 uint8_t *__restrict__ alpha) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long *a = accum + 4 * p;
        unsigned long long cnt = a[3];
        if (cnt > 0) {
            double denom = dmul((double)cnt, 255.0);
            rgb[3 * p + 0] = __double2float_rn(ddiv((double)a[0], denom));
            rgb[3 * p + 1] = __double2float_rn(ddiv((double)a[1], denom));
            rgb[3 * p + 2] = __double2float_rn(ddiv((double)a[2], denom));
            depth[p] = __double2float_rn(minz[p]);
            alpha[p] = 1;
        } else {
            rgb[3 * p + 0] = rgb[3 * p + 1] = rgb[3 * p + 2] = 0.0f;
            depth[p] = 0.0f;
            alpha[p] = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// (ii) fast path: warp tiles over the cell-major scan
// ---------------------------------------------------------------------------

struct SceneArgs {
    const float *pos;
    const uint8_t *col;
    int64_t n;
    const int64_t *occ_off;
    const int32_t *tile_c0;
    const int32_t *tile_c1;
    int64_t n_tiles;
};

__device__ __forceinline__ bool point_kept(const SceneArgs &s, const uint32_t *__restrict__ bits,
                                           int c0, int c1, int64_t i) {
    int lo = c0, hi = c1;  // largest j in [c0,c1] with occ_off[j] <= i
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(s.occ_off + mid) <= i) lo = mid; else hi = mid - 1;
    }
    return (__ldg(bits + (lo >> 5)) >> (lo & 31)) & 1u;
}

__global__ void k_zero_count(uint32_t *__restrict__ count) {
    pdl_wait();
    if (threadIdx.x == 0) *count = 0u;
    pdl_trigger();
}

// Work list of the frame: one u32 per non-culled warp tile, bit 31 = mixed
// (some of its cells culled).  One thread per tile, warp-aggregated append;
// list order is irrelevant (both passes are order-free reductions).
constexpr uint32_t kMixed = 0x80000000u;

__global__ void __launch_bounds__(256) k_tile_list(SceneArgs s, const uint32_t *__restrict__ bits,
                                                   uint32_t *__restrict__ list,
                                                   uint32_t *__restrict__ count) {
    // one list append (atomicAdd) per CTA and 256 tiles, not per warp: the
    // counter is a single address, so per-warp appends serialise in L2
    __shared__ uint32_t wcount[8], cta_off;
    pdl_wait();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < s.n_tiles;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = base + threadIdx.x;
        bool keep_any = false, cull_any = false;
        if (t < s.n_tiles) {
            const int c0 = __ldg(s.tile_c0 + t), c1 = __ldg(s.tile_c1 + t);
            for (int j = c0; j <= c1; ++j) {
                const bool k = (__ldg(bits + (j >> 5)) >> (j & 31)) & 1u;
                keep_any |= k;
                cull_any |= !k;
            }
        }
        const uint32_t vote = __ballot_sync(0xffffffffu, keep_any);
        if (lane == 0) wcount[wid] = (uint32_t)__popc(vote);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < 8; ++w) {
                const uint32_t c = wcount[w];
                wcount[w] = tot;  // exclusive warp offsets
                tot += c;
            }
            cta_off = tot ? atomicAdd(count, tot) : 0u;
        }
        __syncthreads();
        if (keep_any) {
            const uint32_t pos = cta_off + wcount[wid] + __popc(vote & ((1u << lane) - 1u));
            LS_ASSERT(pos < (uint32_t)s.n_tiles);
            list[pos] = (uint32_t)t | (cull_any ? kMixed : 0u);
        }
        __syncthreads();  // wcount / cta_off are rewritten by the next iteration
    }
    pdl_trigger();
}

// Loads the lane's 4 points (xyz) -- vectorised when the group is complete.
__device__ __forceinline__ int load_points(const SceneArgs &s, int64_t base, float (&P)[12]) {
    if (base + 4 <= s.n) {
        const float4 *p4 = reinterpret_cast<const float4 *>(s.pos + 3 * base);
        float4 a = __ldg(p4), b = __ldg(p4 + 1), c = __ldg(p4 + 2);
        P[0] = a.x; P[1] = a.y; P[2] = a.z; P[3] = a.w;
        P[4] = b.x; P[5] = b.y; P[6] = b.z; P[7] = b.w;
        P[8] = c.x; P[9] = c.y; P[10] = c.z; P[11] = c.w;
        return 4;
    }
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < s.n) {
            P[3 * k] = __ldg(s.pos + 3 * (base + k));
            P[3 * k + 1] = __ldg(s.pos + 3 * (base + k) + 1);
            P[3 * k + 2] = __ldg(s.pos + 3 * (base + k) + 2);
            cnt = k + 1;
        } else {
            P[3 * k] = P[3 * k + 1] = P[3 * k + 2] = 0.0f;
        }
    }
    return cnt;
}

__device__ __forceinline__ void load_colors(const SceneArgs &s, int64_t base, int cnt,
                                            uint32_t (&W)[3]) {
    if (cnt == 4) {
        const uint32_t *c4 = reinterpret_cast<const uint32_t *>(s.col + 3 * base);
        W[0] = __ldg(c4);
        W[1] = __ldg(c4 + 1);
        W[2] = __ldg(c4 + 2);
        return;
    }
    W[0] = W[1] = W[2] = 0u;
    for (int b = 0; b < 3 * cnt; ++b) W[b >> 2] |= (uint32_t)__ldg(s.col + 3 * base + b) << (8 * (b & 3));
}

__device__ __forceinline__ uint32_t color_byte(const uint32_t (&W)[3], int b) {
    return (W[b >> 2] >> (8 * (b & 3))) & 0xffu;
}

__device__ __forceinline__ uint32_t color_byte3(uint3 W, int b) {
    const uint32_t w = (b >> 2) == 0 ? W.x : ((b >> 2) == 1 ? W.y : W.z);
    return (w >> (8 * (b & 3))) & 0xffu;
}

__device__ __forceinline__ void red_min_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// {r, g, b, 1} into a pixel's f32 accumulator: one 16 B vector reduction.
__device__ __forceinline__ void red_add_v4f32(float *p, float r, float g, float b) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(r),
                 "f"(g), "f"(b), "f"(1.0f)
                 : "memory");
}

// Iterates the frame's work items (the work list when culling, every tile
// otherwise) through a per-warp ring of S shared-memory stages: lane 0 issues
// bulk async copies (TMA engine, cp.async.bulk) of the tile's xyz (1536 B)
// -- plus its rgb (384 B) for pass 2 -- into a stage, completion tracked by
// the stage's mbarrier, S-1 items ahead of the one being processed.  Lanes
// read their 4 points as 3 x LDS.128 (48 B stride) and colours as 3 x LDS.32
// (12 B stride), both bank-conflict free.  The scan's last, partial tile (and
// rgb of a scene whose colour base is not 16 B aligned) is read from global
// memory.  The ring is kept small (2 stages): the per-pixel minz gathers of
// both passes live off the L1 that the rest of the SM's 256 KB provides.
constexpr int kPassWarps = 8;  // 256-thread CTAs
constexpr int kPosBytes = LS_TILE_POINTS * 12, kColBytes = LS_TILE_POINTS * 3;
// [128 x u32 pixel][128 x depth rounded down: f32, or f16 with LS_CACHE_Z16 (A/B)]
#ifndef LS_CACHE_Z16
#define LS_CACHE_Z16 1
#endif
constexpr int kCacheZBytes = LS_CACHE_Z16 ? 2 : 4;
constexpr int kCacheBytes = LS_TILE_POINTS * (4 + kCacheZBytes);

// A lane's 4 depth records: RD of the f64 camera depth in the cache's format
__device__ __forceinline__ void cache_put_z(uint32_t *blk, int lane, const double (&zc)[4]) {
    float f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = __double2float_rd(zc[k]);
    if constexpr (LS_CACHE_Z16) {
        // RD_f16(RD_f32(z)) = RD_f16(z): f16 values are f32 values
        uint32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __half_as_ushort(__float2half_rd(f[k]));
        reinterpret_cast<uint2 *>(blk + LS_TILE_POINTS)[lane] =
            make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
    } else {
        reinterpret_cast<float4 *>(blk + LS_TILE_POINTS)[lane] = make_float4(f[0], f[1], f[2], f[3]);
    }
}

// ... and back: zlo <= z < znext (znext: the format's next value up, inf past
// its largest finite one)
__device__ __forceinline__ void cache_get_z(const void *zbase, int lane, bool streaming,
                                            float (&zlo)[4], float (&znext)[4]) {
    if constexpr (LS_CACHE_Z16) {
        const uint2 *q = reinterpret_cast<const uint2 *>(zbase) + lane;
        const uint2 v = streaming ? __ldcs(q) : *q;
        const uint32_t h[4] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            zlo[k] = __half2float(__ushort_as_half((unsigned short)h[k]));
            znext[k] = __half2float(__ushort_as_half((unsigned short)(h[k] + 1u)));
        }
    } else {
        const float4 *q = reinterpret_cast<const float4 *>(zbase) + lane;
        const float4 v = streaming ? __ldcs(q) : *q;
        const float z[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            zlo[k] = z[k];
            znext[k] = __int_as_float(__float_as_int(z[k]) + 1);
        }
    }
}
// kXyz: pass 1 | kXyzRgb: pass 2 recomputing | kCacheRgb: pass 2 from the cache
// | kRgb: colours only (multi-view pass 2, whose per-view cache blocks are read
// straight from global memory)
enum RingMode { kXyz = 0, kXyzRgb = 1, kCacheRgb = 2, kRgb = 3 };

template <int S, int MODE>
struct TileRing {
    static constexpr int kMain = MODE == kCacheRgb ? kCacheBytes : (MODE == kRgb ? 0 : kPosBytes);
    static constexpr int kStage = kMain + (MODE == kXyz ? 0 : kColBytes);
    static constexpr size_t kBytes = (size_t)kPassWarps * S * (kStage + 8);  // stages + mbarriers
};

// The scan / cache streams of the passes are read once per frame: tag them
// L2 evict-first so they do not displace the per-pixel minz / accumulator
// lines (~50 MB at 1080p) that every candidate's gather and atomic hits.
// LS_PASS_L2HINT=0 (A/B) drops the hint.
__device__ __forceinline__ uint64_t stream_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
#ifdef LS_NO_PASS_L2HINT
    (void)policy;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(umma::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(umma::smem_u32(bar))
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(umma::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(umma::smem_u32(bar)), "l"(policy)
        : "memory");
#endif
}

// What the body of a pass sees for one work item.
struct Item {
    uint32_t e;         // work-list entry (tile | kMixed)
    int64_t index;      // position in the work list (the item's cache block)
    int64_t base;       // first point of this lane
    bool full;          // complete tile (all 128 points exist)
    const uint8_t *st;  // the item's smem stage
};

template <int S, int MODE, typename F>
__device__ __forceinline__ void for_each_item(const SceneArgs &s, const uint32_t *__restrict__ list,
                                              const uint32_t *__restrict__ count,
                                              const uint32_t *__restrict__ cache, F &&body) {
    using R = TileRing<S, MODE>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t *ring = smem + (size_t)wib * S * R::kStage;
    uint64_t *bars =
        reinterpret_cast<uint64_t *>(smem + (size_t)kPassWarps * S * R::kStage) + wib * S;
    // Item bookkeeping in 32-bit arithmetic: scenes hold < 2^38 points, so tile
    // indices, work-list positions and per-warp counts are < 2^31 (scene_ok).
    const int w0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    const int n_items = list ? (int)__ldg(count) : (int)s.n_tiles;
    if (w0 >= n_items) return;
    const int nj = (n_items - w0 + nw - 1) / nw;  // this warp's items
    const bool col_bulk = MODE != kXyz && (reinterpret_cast<uintptr_t>(s.col) & 15) == 0;
    const uint32_t n_full = (uint32_t)(s.n / LS_TILE_POINTS);  // tiles below hold 128 points
    auto full = [&](uint32_t tile) { return tile < n_full; };
    // Work-list entries of items [32b, 32b+32) live one per lane (ecur), the
    // next 32 in enext, so the issuing lane never waits on a list load.
    auto entry_batch = [&](int b) -> uint32_t {
        const int j = 32 * b + lane;
        if (!list) return (uint32_t)(w0 + j * nw);
        return j < nj ? __ldg(list + w0 + j * nw) : 0u;
    };
    uint32_t ecur = entry_batch(0), enext = entry_batch(1), eprev = 0u;
    int ebatch = 0;
    auto entry = [&](int j) -> uint32_t {  // warp-collective, j non-decreasing
        if ((j >> 5) != ebatch) {
            eprev = ecur;
            ecur = enext;
            ++ebatch;
            enext = entry_batch(ebatch + 1);
        }
        return __shfl_sync(0xffffffffu, ecur, j & 31);
    };
    // the entry of an item up to S - 1 < 32 positions behind the last entry()
    // call (its batch is the current or the previous one)
    auto entry_back = [&](int j) -> uint32_t {
        return __shfl_sync(0xffffffffu, (j >> 5) == ebatch ? ecur : eprev, j & 31);
    };
    const uint64_t pol = stream_policy();
    auto issue = [&](uint32_t e, int j, int q) {  // lane 0 only
        const uint32_t tile = e & ~kMixed;
        const bool f = full(tile);
        // the cache block is always complete (pass 1 writes all 128 slots)
        const bool rgb = MODE != kXyz && f && col_bulk;
        if ((!f && MODE != kCacheRgb) || (MODE == kRgb && !rgb)) {
            umma::mbar_arrive(&bars[q]);
            return;
        }
        umma::mbar_expect_tx(&bars[q], R::kMain + (rgb ? kColBytes : 0));
        uint8_t *dst = ring + q * R::kStage;
        if (MODE == kCacheRgb)
            bulk_g2s(dst, cache + (size_t)(uint32_t)(w0 + j * nw) * (kCacheBytes / 4), kCacheBytes,
                     &bars[q], pol);
        else if (MODE != kRgb)
            bulk_g2s(dst, s.pos + (size_t)tile * (3 * LS_TILE_POINTS), kPosBytes, &bars[q], pol);
        if (rgb)
            bulk_g2s(dst + R::kMain, s.col + (size_t)tile * (3 * LS_TILE_POINTS), kColBytes,
                     &bars[q], pol);
    };
    if (lane == 0) {
        for (int q = 0; q < S; ++q) umma::mbar_init(&bars[q], 1);
        umma::fence_barrier_init();
    }
    for (int q = 0; q < S && q < nj; ++q) {
        const uint32_t e = entry(q);
        if (lane == 0) issue(e, q, q);
    }
    __syncwarp();
    int q = 0;
    uint32_t ph = 0;
    uint32_t index = (uint32_t)w0;  // work-list position of item j: w0 + j * nw
    for (int j = 0; j < nj; ++j, index += (uint32_t)nw) {
        umma::mbar_wait_spin(&bars[q], ph);
        Item it;
        it.e = entry_back(j);
        it.index = index;
        const uint32_t tile = it.e & ~kMixed;
        it.base = (int64_t)tile * LS_TILE_POINTS + 4 * lane;
        it.full = full(tile);
        it.st = ring + q * R::kStage;
        uint3 W = make_uint3(0u, 0u, 0u);  // the lane's 12 colour bytes (by value)
        if (MODE != kXyz) {
            if (it.full && col_bulk) {
                const uint32_t *c4 = reinterpret_cast<const uint32_t *>(it.st + R::kMain) + 3 * lane;
                W = make_uint3(c4[0], c4[1], c4[2]);
            } else {
                uint32_t w3[3];
                const int64_t rem = s.n - it.base;
                load_colors(s, it.base, rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0), w3);
                W = make_uint3(w3[0], w3[1], w3[2]);
            }
        }
        body(it, W);
        if (j + S < nj) {
            const uint32_t en = entry(j + S);
            __syncwarp();
            if (lane == 0) {
                // the lanes' generic-proxy reads of stage q precede the async refill
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(en, j + S, q);
            }
        }
        if (++q == S) {
            q = 0;
            ph ^= 1u;
        }
    }
}

// The lane's 4 points of an item: from the stage when the tile is complete.
__device__ __forceinline__ int item_points(const SceneArgs &s, const Item &it, float (&P)[12]) {
    if (!it.full) return load_points(s, it.base, P);
    const int lane = threadIdx.x & 31;
    const float4 *p4 = reinterpret_cast<const float4 *>(it.st) + 3 * lane;
    const float4 a = p4[0], b = p4[1], c = p4[2];
    P[0] = a.x; P[1] = a.y; P[2] = a.z; P[3] = a.w;
    P[4] = b.x; P[5] = b.y; P[6] = b.z; P[7] = b.w;
    P[8] = c.x; P[9] = c.y; P[10] = c.z; P[11] = c.w;
    return 4;
}

// Culled points of a mixed tile drop out (pix = -1).
__device__ __forceinline__ void drop_culled(const SceneArgs &s, const uint32_t *__restrict__ bits,
                                            const Item &it, int64_t (&pix)[4]) {
    if (!(it.e & kMixed)) return;
    const int64_t tile = it.e & ~kMixed;
    const int c0 = __ldg(s.tile_c0 + tile), c1 = __ldg(s.tile_c1 + tile);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (pix[k] >= 0 && !point_kept(s, bits, c0, c1, it.base + k)) pix[k] = -1;
}

// ---- same-pixel merging inside a lane (pass 2) ---------------------------
// A lane's 4 points are consecutive in the Morton-ordered scan; above ~1
// point per pixel they often share a pixel.  Folding a later point into an
// earlier one on the same pixel is exact (integer colour sums) and saves its
// vector atomic.  (Measured and dropped: the same fold for pass 1's minimum,
// and cross-lane grouping with match.any -- both cost more than they saved.)
__device__ __forceinline__ void merge_lane_sum(int64_t (&pix)[4], uint32_t (&sum)[4][4]) {
#pragma unroll
    for (int k = 1; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < k; ++j)
            if (pix[k] >= 0 && pix[k] == pix[j]) {
#pragma unroll
                for (int c = 0; c < 4; ++c) sum[j][c] += sum[k][c];
                pix[k] = -1;
            }
}

// {r, g, b, n} into a pixel's f32 accumulator: one 16 B vector reduction.
__device__ __forceinline__ void red_add_v4c(float *p, float r, float g, float b, float n) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(r),
                 "f"(g), "f"(b), "f"(n)
                 : "memory");
}

constexpr int kPass1Stages = 2, kPass2Stages = 2;
constexpr uint32_t kNoPixel = 0xFFFFFFFFu;
constexpr size_t kSmem1 = TileRing<kPass1Stages, kXyz>::kBytes;
constexpr size_t kSmem2 = TileRing<kPass2Stages, kXyzRgb>::kBytes;
constexpr size_t kSmem2c = TileRing<kPass2Stages, kCacheRgb>::kBytes;

// Pass 1: per-pixel minimum depth.  A (possibly stale) L1 read of the pixel's
// current minimum filters out points that cannot improve it before the atomic.
// With a cache, every slot's pixel (kNoPixel when rejected) and its depth
// rounded toward -inf to f32 are also recorded, one 1 KB block per work item.
__global__ void __launch_bounds__(256) k_frame_pass1(SceneArgs s, ProjCam c,
                                                     const uint32_t *__restrict__ bits,
                                                     const uint32_t *__restrict__ list,
                                                     const uint32_t *__restrict__ count,
                                                     unsigned long long *__restrict__ minz,
                                                     uint32_t *__restrict__ cache) {
    pdl_wait();
    for_each_item<kPass1Stages, kXyz>(s, list, count, nullptr, [&](const Item &it, uint3) {
        float P[12];
        const int cnt = item_points(s, it, P);
        int64_t pix[4];
        double zc[4];
        project4(P, cnt, c, pix, zc);
        drop_culled(s, bits, it, pix);
        if (cache) {
            const int lane = threadIdx.x & 31;
            uint32_t *blk = cache + it.index * (kCacheBytes / 4);
            reinterpret_cast<uint4 *>(blk)[lane] =
                make_uint4(pix[0] >= 0 ? (uint32_t)pix[0] : kNoPixel,
                           pix[1] >= 0 ? (uint32_t)pix[1] : kNoPixel,
                           pix[2] >= 0 ? (uint32_t)pix[2] : kNoPixel,
                           pix[3] >= 0 ? (uint32_t)pix[3] : kNoPixel);
            cache_put_z(blk, lane, zc);
        }
        unsigned long long key[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) key[k] = (unsigned long long)__double_as_longlong(zc[k]);
        unsigned long long cur[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            cur[k] = pix[k] >= 0 ? __ldca(minz + pix[k]) : 0ull;  // stale L1 is safe: min only decreases
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            LS_ASSERT(pix[k] < c.w * c.h);
            if (pix[k] >= 0 && key[k] < cur[k]) red_min_u64(minz + pix[k], key[k]);
        }
    });
    pdl_trigger();
}

// Pass 1 with 32-bit pixel indices (frames with W*H < 2^32 - 1).
__device__ __forceinline__ void drop_culled_u32(const SceneArgs &s,
                                                const uint32_t *__restrict__ bits,
                                                const Item &it, uint32_t (&pix)[4]) {
    if (!(it.e & kMixed)) return;
    const int64_t tile = it.e & ~kMixed;
    const int c0 = __ldg(s.tile_c0 + tile), c1 = __ldg(s.tile_c1 + tile);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (pix[k] != kNoPixel && !point_kept(s, bits, c0, c1, it.base + k)) pix[k] = kNoPixel;
}

__global__ void __launch_bounds__(256) k_frame_pass1_u32(SceneArgs s, ProjCam c,
                                                         const uint32_t *__restrict__ bits,
                                                         const uint32_t *__restrict__ list,
                                                         const uint32_t *__restrict__ count,
                                                         unsigned long long *__restrict__ minz,
                                                         uint32_t *__restrict__ cache) {
    pdl_wait();
    for_each_item<kPass1Stages, kXyz>(s, list, count, nullptr, [&](const Item &it, uint3) {
        float P[12];
        const int cnt = item_points(s, it, P);
        uint32_t pix[4];
        double zc[4];
        project4_u32(P, cnt, c, pix, zc);
        drop_culled_u32(s, bits, it, pix);
        if (cache) {
            const int lane = threadIdx.x & 31;
            uint32_t *blk = cache + it.index * (kCacheBytes / 4);
            reinterpret_cast<uint4 *>(blk)[lane] = make_uint4(pix[0], pix[1], pix[2], pix[3]);
            cache_put_z(blk, lane, zc);
        }
        unsigned long long cur[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            cur[k] = pix[k] != kNoPixel ? __ldca(minz + pix[k]) : 0ull;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned long long key = (unsigned long long)__double_as_longlong(zc[k]);
#ifdef LS_EXP_NO_RED1  // timing experiment only (scripts/exp): wrong frames
            if (key == 1ull)
#endif
            if (pix[k] != kNoPixel && key < cur[k]) {
                LS_ASSERT((int64_t)pix[k] < c.w * c.h);
                red_min_u64(minz + pix[k], key);
            }
        }
    });
    pdl_trigger();
}

// Pass 2, recompute mode: pixel and depth again from the points.
__global__ void __launch_bounds__(256) k_frame_pass2(SceneArgs s, ProjCam c,
                                                     const uint32_t *__restrict__ bits,
                                                     const uint32_t *__restrict__ list,
                                                     const uint32_t *__restrict__ count, double ope,
                                                     const unsigned long long *__restrict__ minz,
                                                     float *__restrict__ acc) {
    pdl_wait();
    for_each_item<kPass2Stages, kXyzRgb>(s, list, count, nullptr, [&](const Item &it, uint3 W) {
        float P[12];
        const int cnt = item_points(s, it, P);
        int64_t pix[4];
        double zc[4];
        project4(P, cnt, c, pix, zc);
        drop_culled(s, bits, it, pix);
        unsigned long long m[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            m[k] = pix[k] >= 0 ? __ldg(minz + pix[k]) : 0ull;
        uint32_t sum[4][4];  // r, g, b, count of the kept points
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (pix[k] >= 0 && !(zc[k] <= dmul(__longlong_as_double((long long)m[k]), ope)))
                pix[k] = -1;
            sum[k][0] = color_byte3(W, 3 * k);
            sum[k][1] = color_byte3(W, 3 * k + 1);
            sum[k][2] = color_byte3(W, 3 * k + 2);
            sum[k][3] = 1u;
        }
        merge_lane_sum(pix, sum);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (pix[k] >= 0) {
                LS_ASSERT(pix[k] < c.w * c.h);
                red_add_v4c(acc + 4 * pix[k], (float)sum[k][0], (float)sum[k][1], (float)sum[k][2],
                            (float)sum[k][3]);
            }
    });
    pdl_trigger();
}

// Pass 2, cached mode: no projection (pass 2 is instruction-issue bound once
// the scan is Morton ordered).  With T = minz * (1 + eps) in f64 and the
// cached zlo = RD_f32(zc) <= zc <= nextup(zlo): nextup(zlo) <= T keeps,
// zlo > T drops, and only a slot within one f32 ulp of T re-derives its
// exact f64 depth from the point -- the same decision as re-projecting.
__global__ void __launch_bounds__(256) k_frame_pass2_cached(SceneArgs s, ProjCam c,
                                                            const uint32_t *__restrict__ list,
                                                            const uint32_t *__restrict__ count,
                                                            const uint32_t *__restrict__ cache,
                                                            double ope,
                                                            const unsigned long long *__restrict__ minz,
                                                            float *__restrict__ acc) {
    const int lane = threadIdx.x & 31;
    pdl_wait();
    for_each_item<kPass2Stages, kCacheRgb>(s, list, count, cache, [&](const Item &it, uint3 W) {
        const uint4 pw = reinterpret_cast<const uint4 *>(it.st)[lane];
        float zlo[4], znext[4];
        cache_get_z(it.st + 4 * LS_TILE_POINTS, lane, false, zlo, znext);
        uint32_t pix[4] = {pw.x, pw.y, pw.z, pw.w};
        unsigned long long m[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) m[k] = pix[k] != kNoPixel ? __ldg(minz + pix[k]) : 0ull;
        uint32_t sum[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (pix[k] != kNoPixel) {
                const double t = dmul(__longlong_as_double((long long)m[k]), ope);
                // for a float z: (double)z <= T  <=>  z <= RD_f32(T), and
                // z > T  <=>  z > RD_f32(T) (no float lies strictly between
                // RD(T) and RU(T)), so both tests run in f32 against one rounding
                const float trd = __double2float_rd(t);
                bool keep = znext[k] <= trd;
                if (!keep && !(zlo[k] > trd)) {  // within one ulp: exact depth
                    const float *p = s.pos + 3 * (it.base + k);
                    const double x = (double)__ldg(p), y = (double)__ldg(p + 1),
                                 z = (double)__ldg(p + 2);
                    const double zc =
                        dadd(dadd(dadd(dmul(c.r[6], x), dmul(c.r[7], y)), dmul(c.r[8], z)), c.t[2]);
                    keep = zc <= t;
                }
                if (!keep) pix[k] = kNoPixel;
            }
            sum[k][0] = color_byte3(W, 3 * k);
            sum[k][1] = color_byte3(W, 3 * k + 1);
            sum[k][2] = color_byte3(W, 3 * k + 2);
            sum[k][3] = 1u;
        }
        // fold the lane's same-pixel points (integer sums: exact)
#pragma unroll
        for (int k = 1; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < k; ++j)
                if (pix[k] != kNoPixel && pix[k] == pix[j]) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) sum[j][q] += sum[k][q];
                    pix[k] = kNoPixel;
                }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (pix[k] != kNoPixel) {
                LS_ASSERT((int64_t)pix[k] < c.w * c.h);
#ifdef LS_EXP_NO_RED2  // timing experiment only (scripts/exp): wrong frames
                if (sum[k][3] == 1000u)
#endif
                red_add_v4c(acc + 4 * (size_t)pix[k], (float)sum[k][0], (float)sum[k][1],
                            (float)sum[k][2], (float)sum[k][3]);
            }
    });
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// (iii) multi-view batched passes: one read of the culled
// scan feeds up to LS_MAX_VIEWS views.  Each view's arithmetic, culling and
// reductions are exactly those of the single-view passes (render.py:84-143
// run once per view), so every view's frame is bit-identical to rendering it
// alone; what is shared is the tile stream (xyz, rgb, work list).
// ---------------------------------------------------------------------------

struct ViewCams {
    ProjCam c[LS_MAX_VIEWS];
};

// Work list over the union of the views' keep bits, plus a status word per
// entry: bit 2v = view v keeps some cell of the tile, bit 2v+1 = view v also
// culls some cell of it (its points then need the per-point cell test).
__global__ void __launch_bounds__(256) k_tile_list_views(SceneArgs s,
                                                         const uint32_t *__restrict__ bits,
                                                         int64_t words, int nv,
                                                         uint32_t *__restrict__ list,
                                                         uint32_t *__restrict__ status,
                                                         uint32_t *__restrict__ count) {
    __shared__ uint32_t wcount[8], cta_off;  // one append per CTA (see k_tile_list)
    pdl_wait();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < s.n_tiles;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = base + threadIdx.x;
        uint32_t st = 0u;
        if (t < s.n_tiles) {
            const int c0 = __ldg(s.tile_c0 + t), c1 = __ldg(s.tile_c1 + t);
            for (int v = 0; v < nv; ++v) {
                const uint32_t *b = bits + v * words;
                bool keep_any = false, cull_any = false;
                for (int j = c0; j <= c1; ++j) {
                    const bool k = (__ldg(b + (j >> 5)) >> (j & 31)) & 1u;
                    keep_any |= k;
                    cull_any |= !k;
                }
                if (keep_any) st |= (cull_any ? 3u : 1u) << (2 * v);
            }
        }
        const uint32_t vote = __ballot_sync(0xffffffffu, st != 0u);
        if (lane == 0) wcount[wid] = (uint32_t)__popc(vote);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < 8; ++w) {
                const uint32_t c = wcount[w];
                wcount[w] = tot;
                tot += c;
            }
            cta_off = tot ? atomicAdd(count, tot) : 0u;
        }
        __syncthreads();
        if (st != 0u) {
            const uint32_t at = cta_off + wcount[wid] + __popc(vote & ((1u << lane) - 1u));
            list[at] = (uint32_t)t;
            status[at] = st;
        }
        __syncthreads();
    }
    pdl_trigger();
}

// Status word of an item: every view keeps every point when there is no cull.
__device__ __forceinline__ uint32_t item_status(const uint32_t *__restrict__ status,
                                                const Item &it) {
    return status ? __ldg(status + it.index) : 0x5555u;
}

// drop_culled against one view's keep bits (the tile straddles a culled cell).
__device__ __forceinline__ void drop_culled_view(const SceneArgs &s,
                                                 const uint32_t *__restrict__ bits,
                                                 const Item &it, int64_t (&pix)[4]) {
    const int64_t tile = it.e & ~kMixed;
    const int c0 = __ldg(s.tile_c0 + tile), c1 = __ldg(s.tile_c1 + tile);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (pix[k] >= 0 && !point_kept(s, bits, c0, c1, it.base + k)) pix[k] = -1;
}

// The multi-view passes are instantiated for NV = 1, 2, 4, 8 view slots
// (slots >= n_views carry status 0); the view loop is unrolled so each view's
// camera stays constant-bank operands, exactly like the single-view passes.
// With a cache, view v of work item i owns the 1 KB block i * n_views + v
// (pass 1 writes it, pass 2 decides from it: the single-view cache rule).
template <int NV>
__global__ void __launch_bounds__(256, 3) k_frame_pass1_views(
    SceneArgs s, const ViewCams vc, int nv, int64_t npix, const uint32_t *__restrict__ bits,
    int64_t words, const uint32_t *__restrict__ list, const uint32_t *__restrict__ status,
    const uint32_t *__restrict__ count, unsigned long long *__restrict__ minz,
    uint32_t *__restrict__ cache) {
    pdl_wait();
    const uint32_t live = (1u << (2 * nv)) - 1u;
    for_each_item<kPass1Stages, kXyz>(s, list, count, nullptr, [&](const Item &it, uint3) {
        float P[12];
        const int cnt = item_points(s, it, P);
        const uint32_t st = item_status(status, it) & live;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const uint32_t vs = (st >> (2 * v)) & 3u;
            if (vs == 0u) continue;
            int64_t pix[4];
            double zc[4];
            project4(P, cnt, vc.c[v], pix, zc);
            if (vs == 3u) drop_culled_view(s, bits + v * words, it, pix);
            if (cache) {
                const int lane = threadIdx.x & 31;
                uint32_t *blk = cache + (it.index * nv + v) * (kCacheBytes / 4);
                reinterpret_cast<uint4 *>(blk)[lane] =
                    make_uint4(pix[0] >= 0 ? (uint32_t)pix[0] : kNoPixel,
                               pix[1] >= 0 ? (uint32_t)pix[1] : kNoPixel,
                               pix[2] >= 0 ? (uint32_t)pix[2] : kNoPixel,
                               pix[3] >= 0 ? (uint32_t)pix[3] : kNoPixel);
                cache_put_z(blk, lane, zc);
            }
            unsigned long long *mz = minz + v * npix;
            unsigned long long key[4], cur[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) key[k] = (unsigned long long)__double_as_longlong(zc[k]);
#pragma unroll
            for (int k = 0; k < 4; ++k) cur[k] = pix[k] >= 0 ? __ldca(mz + pix[k]) : 0ull;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                LS_ASSERT(pix[k] < npix);
                if (pix[k] >= 0 && key[k] < cur[k]) red_min_u64(mz + pix[k], key[k]);
            }
        }
    });
    pdl_trigger();
}

// Keep decision + lane fold + vector atomics of one view's 4 points (shared
// by both multi-view pass-2 forms).
__device__ __forceinline__ void accumulate4(int64_t (&pix)[4], const uint3 &W, float *a) {
    uint32_t sum[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        sum[k][0] = color_byte3(W, 3 * k);
        sum[k][1] = color_byte3(W, 3 * k + 1);
        sum[k][2] = color_byte3(W, 3 * k + 2);
        sum[k][3] = 1u;
    }
    merge_lane_sum(pix, sum);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (pix[k] >= 0)
            red_add_v4c(a + 4 * pix[k], (float)sum[k][0], (float)sum[k][1], (float)sum[k][2],
                        (float)sum[k][3]);
}

template <int NV>
__global__ void __launch_bounds__(256, 3) k_frame_pass2_views(
    SceneArgs s, const ViewCams vc, int nv, int64_t npix, const uint32_t *__restrict__ bits,
    int64_t words, const uint32_t *__restrict__ list, const uint32_t *__restrict__ status,
    const uint32_t *__restrict__ count, double ope, const unsigned long long *__restrict__ minz,
    float *__restrict__ acc) {
    pdl_wait();
    const uint32_t live = (1u << (2 * nv)) - 1u;
    for_each_item<kPass2Stages, kXyzRgb>(s, list, count, nullptr, [&](const Item &it, uint3 W) {
        float P[12];
        const int cnt = item_points(s, it, P);
        const uint32_t st = item_status(status, it) & live;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const uint32_t vs = (st >> (2 * v)) & 3u;
            if (vs == 0u) continue;
            int64_t pix[4];
            double zc[4];
            project4(P, cnt, vc.c[v], pix, zc);
            if (vs == 3u) drop_culled_view(s, bits + v * words, it, pix);
            const unsigned long long *mz = minz + v * npix;
            unsigned long long m[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) m[k] = pix[k] >= 0 ? __ldg(mz + pix[k]) : 0ull;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (pix[k] >= 0 && !(zc[k] <= dmul(__longlong_as_double((long long)m[k]), ope)))
                    pix[k] = -1;
            accumulate4(pix, W, acc + 4 * v * npix);
        }
    });
    pdl_trigger();
}

// Pass 2 from the per-view cache (k_frame_pass2_cached's rule per view): the
// ring carries only colours; a view's 1 KB block is one coalesced 16 B load
// per lane for pixels and one for depths.
template <int NV>
__global__ void __launch_bounds__(256) k_frame_pass2_views_cached(
    SceneArgs s, const ViewCams vc, int nv, int64_t npix, const uint32_t *__restrict__ list,
    const uint32_t *__restrict__ status, const uint32_t *__restrict__ count,
    const uint32_t *__restrict__ cache, double ope, const unsigned long long *__restrict__ minz,
    float *__restrict__ acc) {
    const int lane = threadIdx.x & 31;
    pdl_wait();
    const uint32_t live = (1u << (2 * nv)) - 1u;
    for_each_item<kPass2Stages, kRgb>(s, list, count, nullptr, [&](const Item &it, uint3 W) {
        const uint32_t st = item_status(status, it) & live;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if (((st >> (2 * v)) & 3u) == 0u) continue;
            const uint32_t *blk = cache + (it.index * nv + v) * (kCacheBytes / 4);
            const uint4 pw = __ldcs(reinterpret_cast<const uint4 *>(blk) + lane);
            float zlo[4], znext[4];
            cache_get_z(blk + LS_TILE_POINTS, lane, true, zlo, znext);
            const uint32_t pc[4] = {pw.x, pw.y, pw.z, pw.w};
            const unsigned long long *mz = minz + v * npix;
            unsigned long long m[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) m[k] = pc[k] != kNoPixel ? __ldg(mz + pc[k]) : 0ull;
            int64_t pix[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                pix[k] = -1;
                if (pc[k] == kNoPixel) continue;
                const double t = dmul(__longlong_as_double((long long)m[k]), ope);
                const float trd = __double2float_rd(t);
                bool keep = znext[k] <= trd;
                if (!keep && !(zlo[k] > trd)) {  // within one ulp: exact depth
                    const float *p = s.pos + 3 * (it.base + k);
                    const double x = (double)__ldg(p), y = (double)__ldg(p + 1),
                                 z = (double)__ldg(p + 2);
                    const ProjCam &c = vc.c[v];
                    const double zc =
                        dadd(dadd(dadd(dmul(c.r[6], x), dmul(c.r[7], y)), dmul(c.r[8], z)), c.t[2]);
                    keep = zc <= t;
                }
                if (keep) pix[k] = (int64_t)pc[k];
            }
            accumulate4(pix, W, acc + 4 * v * npix);
        }
    });
    pdl_trigger();
}

// Per-scan: occupied-cell span of every warp tile.
__global__ void k_tile_index(const int64_t *__restrict__ occ_off, int64_t n_occ, int64_t n,
                             int64_t n_tiles, int32_t *__restrict__ c0, int32_t *__restrict__ c1) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t first = t * LS_TILE_POINTS;
        int64_t last = min(first + LS_TILE_POINTS, n) - 1;
        int64_t res[2];
        int64_t q[2] = {first, last};
        for (int e = 0; e < 2; ++e) {
            int64_t lo = 0, hi = n_occ - 1;
            while (lo < hi) {
                int64_t mid = (lo + hi + 1) >> 1;
                if (occ_off[mid] <= q[e]) lo = mid; else hi = mid - 1;
            }
            res[e] = lo;
        }
        c0[t] = (int32_t)res[0];
        c1[t] = (int32_t)res[1];
    }
}

inline SceneArgs scene_args(const ls_scene &s) {
    SceneArgs a;
    a.pos = s.d_positions;
    a.col = s.d_colors;
    a.n = s.n_points;
    a.occ_off = s.d_occ_offsets;
    a.tile_c0 = s.d_tile_c0;
    a.tile_c1 = s.d_tile_c1;
    a.n_tiles = s.n_tiles;
    return a;
}

inline bool camera_ok(const ls_camera *cam) {
    // width/height < 2^31: the frame passes test 0 <= u < W on the low word
    // of u + 2^52 (ls_common.cuh project4)
    return cam && cam->width > 0 && cam->height > 0 && cam->width < (int64_t(1) << 31) &&
           cam->height < (int64_t(1) << 31) && cam->z_near > 0.0 &&
           cam->width * cam->height < (int64_t(1) << 40);
}

// Frame passes: 256-thread CTAs with a dynamic-smem tile ring, exactly as
// many as are co-resident (persistent, grid-stride over the work list; a
// grid of several waves would leave a partial last wave).
static int ring_blocks_per_sm(const void *fn, size_t smem) {
    struct Entry {
        const void *fn;
        int blocks;
    };
    static Entry cache[32];
    static int n = 0;
    static std::mutex mu;  // ABI calls may come from several host threads
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; ++i)
        if (cache[i].fn == fn) return cache[i].blocks;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // half of the unified 256 KB as shared memory: 4 CTAs' rings fit, and the
    // other half stays L1 for the per-pixel minz gathers (measured: leaving the
    // split to the driver shrinks L1 to ~30 KB and costs pass 1 ~60%)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 50);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, 256, smem) != cudaSuccess || b < 1)
        b = 1;
    if (n < 32) cache[n++] = {fn, b};
    return b;
}

template <typename K>
inline int frame_grid(K kernel, size_t smem, int64_t n_tiles) {
    return grid_for(n_tiles * 32, 256, ring_blocks_per_sm((const void *)kernel, smem));
}

}  // namespace ls

using namespace ls;

extern "C" {

size_t ls_ranges_workspace(int64_t n_ranges) { return sizeof(int64_t) * (size_t)(n_ranges + 1); }

int ls_project_min_depth(const float *d_positions, const int64_t *d_starts, const int64_t *d_ends,
                         int64_t n_ranges, const ls_camera *cam, double *d_minz,
                         int64_t *d_pix_cache, double *d_z_cache, void *d_workspace,
                         size_t workspace_bytes, void *stream) {
    if (n_ranges < 0 || !camera_ok(cam) || workspace_bytes < ls_ranges_workspace(n_ranges))
        return LS_EINVAL;
    if (n_ranges == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t *prefix = (int64_t *)d_workspace;
    k_range_prefix<<<1, 1024, 0, st>>>(d_starts, d_ends, n_ranges, prefix);
    LS_LAUNCH_CHECK();
    k_twin_pass1<<<kSmCount * 8, 256, 0, st>>>(d_positions, d_starts, prefix, n_ranges,
                                              make_cam(*cam), (unsigned long long *)d_minz,
                                              d_pix_cache, d_z_cache);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_project_accumulate(const uint8_t *d_colors, const int64_t *d_starts, const int64_t *d_ends,
                          int64_t n_ranges, const int64_t *d_pix_cache, const double *d_z_cache,
                          double eps_rel, const double *d_minz, uint64_t *d_accum,
                          void *d_workspace, size_t workspace_bytes, void *stream) {
    if (n_ranges < 0 || workspace_bytes < ls_ranges_workspace(n_ranges)) return LS_EINVAL;
    if (n_ranges == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t *prefix = (int64_t *)d_workspace;
    k_range_prefix<<<1, 1024, 0, st>>>(d_starts, d_ends, n_ranges, prefix);
    LS_LAUNCH_CHECK();
    const double ope = 1.0 + eps_rel;  // rounded once (_native.pyx:135)
    k_twin_pass2<<<kSmCount * 8, 256, 0, st>>>(d_colors, d_starts, prefix, n_ranges, d_pix_cache,
                                              d_z_cache, ope, d_minz,
                                              (unsigned long long *)d_accum);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_assemble(const double *d_minz, const uint64_t *d_accum, int64_t n_pixels, float *d_rgb,
                float *d_depth, uint8_t *d_alpha, void *stream) {
    if (n_pixels < 0) return LS_EINVAL;
    if (n_pixels == 0) return 0;
    k_assemble_exact<<<grid_for(n_pixels, 256), 256, 0, (cudaStream_t)stream>>>(
        d_minz, (const unsigned long long *)d_accum, n_pixels, d_rgb, d_depth, d_alpha);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_scene_tile_index(const int64_t *d_occ_offsets, int64_t n_occ, int64_t n_points,
                        int32_t *d_tile_c0, int32_t *d_tile_c1, void *stream) {
    if (n_occ <= 0 || n_points <= 0 || n_occ >= (int64_t(1) << 31)) return LS_EINVAL;
    int64_t n_tiles = (n_points + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    k_tile_index<<<grid_for(n_tiles, 256), 256, 0, (cudaStream_t)stream>>>(
        d_occ_offsets, n_occ, n_points, n_tiles, d_tile_c0, d_tile_c1);
    LS_LAUNCH_CHECK();
    return 0;
}

static bool scene_ok(const ls_scene *scene, const uint32_t *d_list) {
    if (!scene || scene->n_points < 0 || scene->n_points >= (int64_t(1) << 38)) return false;
    // the warp-tile passes load xyz as 3 x 16 B and rgb as 3 x 4 B per 4 points
    if ((reinterpret_cast<uintptr_t>(scene->d_positions) & 15) ||
        (reinterpret_cast<uintptr_t>(scene->d_colors) & 3))
        return false;
    if (d_list && (!scene->d_tile_c0 || !scene->d_tile_c1 || !scene->d_occ_offsets)) return false;
    return true;
}

int ls_tile_worklist(const ls_scene *scene, const uint32_t *d_keep_bits, uint32_t *d_list,
                     uint32_t *d_count, void *stream) {
    if (!scene_ok(scene, d_list) || !d_keep_bits || !d_list || !d_count) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    // a one-thread kernel instead of a memset node keeps the PDL chain unbroken
    cudaError_t e = launch_pdl(k_zero_count, dim3(1), dim3(32), 0, st, d_count);
    if (e != cudaSuccess) return (int)e;
    if (scene->n_points == 0) return 0;
    SceneArgs a = scene_args(*scene);
    a.n_tiles = (a.n + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    return (int)launch_pdl(k_tile_list, dim3(grid_for(a.n_tiles, 256, 8)), dim3(256), 0, st, a,
                           d_keep_bits, d_list, d_count);
}

size_t ls_frame_cache_bytes(const ls_scene *scene) {
    if (!scene || scene->n_points <= 0) return 0;
    return (size_t)((scene->n_points + LS_TILE_POINTS - 1) / LS_TILE_POINTS) * kCacheBytes;
}

static bool cache_ok(const ls_camera *cam, const void *d_cache) {
    // u32 pixel slots with kNoPixel reserved; 16 B vector stores / bulk copies
    return !d_cache || (cam->width * cam->height < (int64_t)kNoPixel &&
                        (reinterpret_cast<uintptr_t>(d_cache) & 15) == 0);
}

// LS_PASS1_U32=0 keeps 64-bit pixel indices in pass 1 (A/B measurements).
static bool pass1_u32() {
    static std::atomic<int> v{-1};  // set-once cache, relaxed is enough
    int r = v.load(std::memory_order_relaxed);
    if (r < 0) {
        const char *e = getenv("LS_PASS1_U32");
        r = (e && e[0] == '0') ? 0 : 1;
        v.store(r, std::memory_order_relaxed);
    }
    return r == 1;
}

int ls_frame_pass1(const ls_scene *scene, const uint32_t *d_keep_bits, const uint32_t *d_list,
                   const uint32_t *d_count, const ls_camera *cam, uint64_t *d_minz_bits,
                   uint32_t *d_cache, void *stream) {
    if (!scene_ok(scene, d_list) || !camera_ok(cam) || (d_list && (!d_count || !d_keep_bits)) ||
        !cache_ok(cam, d_cache))
        return LS_EINVAL;
    if (scene->n_points == 0) return 0;
    SceneArgs a = scene_args(*scene);
    a.n_tiles = (a.n + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    if (cam->width * cam->height < (int64_t)kNoPixel && pass1_u32())
        return (int)launch_pdl(k_frame_pass1_u32,
                               dim3(frame_grid(k_frame_pass1_u32, kSmem1, a.n_tiles)), dim3(256),
                               kSmem1, (cudaStream_t)stream, a, make_cam(*cam), d_keep_bits,
                               d_list, d_count, (unsigned long long *)d_minz_bits, d_cache);
    return (int)launch_pdl(k_frame_pass1, dim3(frame_grid(k_frame_pass1, kSmem1, a.n_tiles)),
                           dim3(256), kSmem1, (cudaStream_t)stream, a, make_cam(*cam), d_keep_bits,
                           d_list, d_count, (unsigned long long *)d_minz_bits, d_cache);
}

int ls_frame_pass2(const ls_scene *scene, const uint32_t *d_keep_bits, const uint32_t *d_list,
                   const uint32_t *d_count, const ls_camera *cam, double eps_rel,
                   const uint64_t *d_minz_bits, const uint32_t *d_cache, float *d_accum4,
                   void *stream) {
    if (!scene_ok(scene, d_list) || !camera_ok(cam) || (d_list && (!d_count || !d_keep_bits)) ||
        !cache_ok(cam, d_cache))
        return LS_EINVAL;
    if (scene->n_points == 0) return 0;
    SceneArgs a = scene_args(*scene);
    a.n_tiles = (a.n + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    const double ope = 1.0 + eps_rel;
    if (d_cache)
        return (int)launch_pdl(k_frame_pass2_cached,
                               dim3(frame_grid(k_frame_pass2_cached, kSmem2c, a.n_tiles)),
                               dim3(256), kSmem2c, (cudaStream_t)stream, a, make_cam(*cam), d_list,
                               d_count, d_cache, ope, (const unsigned long long *)d_minz_bits,
                               d_accum4);
    return (int)launch_pdl(k_frame_pass2, dim3(frame_grid(k_frame_pass2, kSmem2, a.n_tiles)),
                           dim3(256), kSmem2, (cudaStream_t)stream, a, make_cam(*cam), d_keep_bits,
                           d_list, d_count, ope, (const unsigned long long *)d_minz_bits, d_accum4);
}

int ls_frame_project(const ls_scene *scene, const uint32_t *d_keep_bits, uint32_t *d_list,
                     uint32_t *d_count, const ls_camera *cam, double eps_rel,
                     uint64_t *d_minz_bits, uint32_t *d_cache, float *d_accum4, void *stream) {
    int rc = 0;
    if (d_keep_bits) {
        rc = ls_tile_worklist(scene, d_keep_bits, d_list, d_count, stream);
        if (rc) return rc;
    } else {
        d_list = nullptr;
        d_count = nullptr;
    }
    rc = ls_frame_pass1(scene, d_keep_bits, d_list, d_count, cam, d_minz_bits, d_cache, stream);
    if (rc) return rc;
    return ls_frame_pass2(scene, d_keep_bits, d_list, d_count, cam, eps_rel, d_minz_bits, d_cache,
                          d_accum4, stream);
}

// Re-target a captured frame graph (stream capture of ls_cull +
// ls_tile_worklist + ls_frame_pass1/2 + the rest of the frame) to another
// camera: the k_cull nodes get the new frustum planes and the projection
// pass nodes the new camera, through cudaGraphExecKernelNodeSetParams; every
// other node (work list, assembly, filter, U-Net) is camera-independent.
int ls_frame_graph_set_camera(void *graph, void *graph_exec, const ls_camera *cam,
                              const double h_planes[24]) {
    if (!graph || !graph_exec || !camera_ok(cam) || !h_planes) return LS_EINVAL;
    cudaGraph_t g = (cudaGraph_t)graph;
    cudaGraphExec_t ge = (cudaGraphExec_t)graph_exec;
    size_t n = 0;
    cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
    if (e != cudaSuccess) return (int)e;
    if (n == 0) return LS_EINVAL;
    cudaGraphNode_t nodes[512];
    if (n > 512) return LS_EINVAL;
    e = cudaGraphGetNodes(g, nodes, &n);
    if (e != cudaSuccess) return (int)e;
    const ProjCam pc = make_cam(*cam);
    double planes[24];
    for (int i = 0; i < 24; ++i) planes[i] = h_planes[i];
    // (kernel, its parameter count, the index of its camera / planes argument)
    struct Target {
        const void *fn;
        int nargs, arg;
        const void *val;
    };
    const Target targets[] = {
        {cull_kernel(), 11, cull_planes_arg(), planes},
        {(const void *)k_frame_pass1, 7, 1, &pc},
        {(const void *)k_frame_pass1_u32, 7, 1, &pc},
        {(const void *)k_frame_pass2, 8, 1, &pc},
        {(const void *)k_frame_pass2_cached, 8, 1, &pc},
    };
    int updated = 0;
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess || t != cudaGraphNodeTypeKernel)
            continue;
        cudaKernelNodeParams kp;
        e = cudaGraphKernelNodeGetParams(nodes[i], &kp);
        if (e != cudaSuccess) return (int)e;
        for (const Target &tg : targets) {
            if (kp.func != tg.fn) continue;
            void *args[16];
            for (int a = 0; a < tg.nargs; ++a) args[a] = kp.kernelParams[a];
            args[tg.arg] = const_cast<void *>(tg.val);
            kp.kernelParams = args;
            kp.extra = nullptr;
            e = cudaGraphExecKernelNodeSetParams(ge, nodes[i], &kp);
            if (e != cudaSuccess) return (int)e;
            ++updated;
        }
    }
    return updated >= 1 ? 0 : LS_EINVAL;
}

int ls_tile_worklist_views(const ls_scene *scene, const uint32_t *d_keep_bits,
                           int64_t bits_stride, int32_t n_views, uint32_t *d_list,
                           uint32_t *d_status, uint32_t *d_count, void *stream) {
    if (!scene_ok(scene, d_list) || !d_keep_bits || !d_list || !d_status || !d_count ||
        n_views < 1 || n_views > LS_MAX_VIEWS || bits_stride < (scene->n_occ + 31) / 32)
        return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = launch_pdl(k_zero_count, dim3(1), dim3(32), 0, st, d_count);
    if (e != cudaSuccess) return (int)e;
    if (scene->n_points == 0) return 0;
    SceneArgs a = scene_args(*scene);
    a.n_tiles = (a.n + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    return (int)launch_pdl(k_tile_list_views, dim3(grid_for(a.n_tiles, 256, 8)), dim3(256), 0, st,
                           a, d_keep_bits, bits_stride, (int)n_views, d_list, d_status, d_count);
}

size_t ls_frame_views_cache_bytes(const ls_scene *scene, int32_t n_views) {
    if (n_views < 1 || n_views > LS_MAX_VIEWS) return 0;
    return ls_frame_cache_bytes(scene) * (size_t)n_views;
}

}  // extern "C"

namespace ls {

template <int NV>
static int launch_views(const SceneArgs &a, const ViewCams &vc, int nv, int64_t npix,
                        const uint32_t *bits, int64_t stride, const uint32_t *list,
                        const uint32_t *status, const uint32_t *count, double ope,
                        uint64_t *minz, uint32_t *cache, float *acc, cudaStream_t st) {
    cudaError_t e = launch_pdl(k_frame_pass1_views<NV>,
                               dim3(frame_grid(k_frame_pass1_views<NV>, kSmem1, a.n_tiles)),
                               dim3(256), kSmem1, st, a, vc, nv, npix, bits, stride, list, status,
                               count, (unsigned long long *)minz, cache);
    if (e != cudaSuccess) return (int)e;
    if (cache) {
        constexpr size_t kSm = TileRing<kPass2Stages, kRgb>::kBytes;
        return (int)launch_pdl(k_frame_pass2_views_cached<NV>,
                               dim3(frame_grid(k_frame_pass2_views_cached<NV>, kSm, a.n_tiles)),
                               dim3(256), kSm, st, a, vc, nv, npix, list, status, count,
                               (const uint32_t *)cache, ope, (const unsigned long long *)minz,
                               acc);
    }
    return (int)launch_pdl(k_frame_pass2_views<NV>,
                           dim3(frame_grid(k_frame_pass2_views<NV>, kSmem2, a.n_tiles)),
                           dim3(256), kSmem2, st, a, vc, nv, npix, bits, stride, list, status,
                           count, ope, (const unsigned long long *)minz, acc);
}

}  // namespace ls

extern "C" {

int ls_frame_project_views(const ls_scene *scene, const uint32_t *d_keep_bits,
                           int64_t bits_stride, uint32_t *d_list, uint32_t *d_status,
                           uint32_t *d_count, const ls_camera *cams, int32_t n_views,
                           double eps_rel, uint64_t *d_minz_bits, uint32_t *d_cache,
                           float *d_accum4, void *stream) {
    if (!scene_ok(scene, d_keep_bits ? d_list : nullptr) || !cams || n_views < 1 ||
        n_views > LS_MAX_VIEWS || !d_minz_bits || !d_accum4)
        return LS_EINVAL;
    ViewCams vc;
    for (int v = 0; v < n_views; ++v) {
        if (!camera_ok(cams + v) || cams[v].width != cams[0].width ||
            cams[v].height != cams[0].height || !cache_ok(cams + v, d_cache))
            return LS_EINVAL;
        vc.c[v] = make_cam(cams[v]);
    }
    for (int v = n_views; v < LS_MAX_VIEWS; ++v) vc.c[v] = vc.c[0];
    if (scene->n_points == 0) return 0;
    int rc = 0;
    if (d_keep_bits) {
        rc = ls_tile_worklist_views(scene, d_keep_bits, bits_stride, n_views, d_list, d_status,
                                    d_count, stream);
        if (rc) return rc;
    } else {
        d_list = d_status = d_count = nullptr;
    }
    SceneArgs a = scene_args(*scene);
    a.n_tiles = (a.n + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    const int64_t npix = cams[0].width * cams[0].height;
    const double ope = 1.0 + eps_rel;  // rounded once (_native.pyx:135)
    cudaStream_t st = (cudaStream_t)stream;
    auto go = [&](auto tag) {
        return launch_views<decltype(tag)::value>(a, vc, n_views, npix, d_keep_bits, bits_stride,
                                                  d_list, d_status, d_count, ope, d_minz_bits,
                                                  d_cache, d_accum4, st);
    };
    if (n_views == 1) return go(std::integral_constant<int, 1>());
    if (n_views == 2) return go(std::integral_constant<int, 2>());
    if (n_views <= 4) return go(std::integral_constant<int, 4>());
    return go(std::integral_constant<int, 8>());
}

}  // extern "C"
