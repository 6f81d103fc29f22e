// Per-scan grid build on the device (grid.py:94-128): cell assignment, the
// stable counting sort and the cell-major gathers.
//
// assign_cells is a bit-exact f64 restatement of _native.pyx:19-44.  The stable
// counting sort (_native.pyx:47-68) is a hand-written LSD radix sort of the
// cell ids carrying u32 point indices (stable per pass, hence overall: the
// permutation equals the reference's counting sort), followed by a
// lower-bound pass that materialises cell_offsets.
#include "ls_common.cuh"

namespace ls {

// ---- stable LSD radix sort (8-bit digits) ---------------------------------
// Per pass over a digit: (1) every CTA counts its 4096-key block's digits in
// shared memory and writes them digit-major (hist[digit * n_blocks + block]);
// (2) an exclusive scan of that array gives every (digit, block) its output
// base -- all smaller digits first, then earlier blocks of the same digit;
// (3) every CTA re-reads its block and scatters each key/value to base +
// its rank among the block's keys with the same digit that precede it.  The
// rank is stable by construction: warp w owns the block's w-th 512 keys in
// 16 consecutive 32-key steps; inside a step, lanes with equal digits
// (8 ballots) rank by lane; steps accumulate per-warp digit counters; warps
// are offset by the counts of the warps before them.
constexpr int kSortThreads = 256, kSortPerThread = 16;
constexpr int kSortBlock = kSortThreads * kSortPerThread;  // 4096 keys
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kScanChunk = 4096;

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
    return (uint32_t)(key >> shift) & 0xFFu;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const K *__restrict__ keys, int64_t n,
                                                             int shift, int64_t n_blocks,
                                                             uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += kSortThreads) h[i] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * kSortBlock;
    for (int i = threadIdx.x; i < kSortBlock; i += kSortThreads) {
        const int64_t k = b0 + i;
        if (k < n) atomicAdd(&h[digit_of(keys[k], shift)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += kSortThreads)
        hist[(int64_t)d * n_blocks + blockIdx.x] = h[d];
}

// exclusive scan of a u32 array: per-chunk scan + chunk totals, a scan of
// the totals (one CTA), then the chunk prefixes added back
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *warp_tot,
                                                         uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t incl = x + (wid > 0 ? warp_tot[wid - 1] : 0u);
    total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return incl - v;
}

__global__ void __launch_bounds__(kSortThreads) k_scan_chunks(uint32_t *__restrict__ a, int64_t len,
                                                              uint32_t *__restrict__ totals) {
    __shared__ uint32_t wt[32];
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk;
    uint32_t carry = 0;
    for (int base = 0; base < kScanChunk; base += kSortThreads) {
        const int64_t i = c0 + base + threadIdx.x;
        const uint32_t v = i < len ? a[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(v, wt, tot);
        if (i < len) a[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(kSortThreads) k_scan_totals(uint32_t *__restrict__ totals,
                                                              int64_t m) {
    __shared__ uint32_t wt[32];
    uint32_t carry = 0;
    for (int64_t base = 0; base < m; base += kSortThreads) {
        const int64_t i = base + threadIdx.x;
        const uint32_t v = i < m ? totals[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(v, wt, tot);
        if (i < m) totals[i] = carry + ex;
        carry += tot;
    }
}

__global__ void k_scan_add(uint32_t *__restrict__ a, int64_t len,
                           const uint32_t *__restrict__ totals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] += totals[i / kScanChunk];
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(
    const K *__restrict__ keys, const uint32_t *__restrict__ vals, int64_t n, int shift,
    int64_t n_blocks, const uint32_t *__restrict__ base, K *__restrict__ keys_out,
    uint32_t *__restrict__ vals_out) {
    __shared__ uint32_t cnt[kSortWarps][256];  // per-warp digit counts, then warp offsets
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t k0 = (int64_t)blockIdx.x * kSortBlock + (int64_t)w * (32 * kSortPerThread);
    K key[kSortPerThread];
    uint32_t dig[kSortPerThread], rank[kSortPerThread];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortPerThread; ++j) {
        const int64_t k = k0 + 32 * j + lane;
        const bool ok = k < n;
        key[j] = ok ? keys[k] : K(0);
        const uint32_t d = ok ? digit_of(key[j], shift) : 256u;
        dig[j] = d;
        // lanes holding the same digit (valid lanes only)
        uint32_t peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
        }
        uint32_t r = 0;
        if (ok) {
            r = cnt[w][d] + __popc(peers & lt);
        }
        __syncwarp();
        // the highest peer advances the warp's counter for this digit
        if (ok && (peers >> lane) == 1u) cnt[w][d] += __popc(peers);
        __syncwarp();
        rank[j] = r;
    }
    __syncthreads();
    // warp offsets: exclusive scan over warps, per digit
    for (int d = threadIdx.x; d < 256; d += kSortThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < kSortWarps; ++ww) {
            const uint32_t c = cnt[ww][d];
            cnt[ww][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortPerThread; ++j) {
        const int64_t k = k0 + 32 * j + lane;
        if (k >= n) continue;
        const uint32_t d = dig[j];
        const uint32_t pos = base[(int64_t)d * n_blocks + blockIdx.x] + cnt[w][d] + rank[j];
        keys_out[pos] = key[j];
        vals_out[pos] = vals ? vals[k] : (uint32_t)k;
    }
}

inline size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

inline int64_t sort_blocks(int64_t n) { return (n + kSortBlock - 1) / kSortBlock; }

// scratch of one radix sort: histogram/offsets + chunk totals
inline size_t radix_scratch_bytes(int64_t n) {
    const int64_t len = 256 * sort_blocks(n);
    const int64_t chunks = (len + kScanChunk - 1) / kScanChunk;
    return a256(4 * (size_t)len) + a256(4 * (size_t)chunks);
}

// Stable sort of (keys, u32 values = input positions) on bits [0, end_bit)
// with ping-pong buffers; returns the buffers holding the result.
template <typename K>
int radix_sort(K *keys_a, K *keys_b, uint32_t *vals_a, uint32_t *vals_b, int64_t n, int end_bit,
               void *scratch, cudaStream_t st, K *&keys_res, uint32_t *&vals_res) {
    const int64_t nb = sort_blocks(n);
    const int64_t len = 256 * nb;
    const int64_t chunks = (len + kScanChunk - 1) / kScanChunk;
    uint32_t *hist = (uint32_t *)scratch;
    uint32_t *totals = (uint32_t *)((char *)scratch + a256(4 * (size_t)len));
    K *kbuf[2] = {keys_a, keys_b};
    uint32_t *vbuf[2] = {vals_a, vals_b};
    int cur = 0;
    const uint32_t *vin = nullptr;  // pass 0 takes the input positions as values
    for (int shift = 0; shift < end_bit; shift += 8) {
        k_radix_hist<K><<<(unsigned)nb, kSortThreads, 0, st>>>(kbuf[cur], n, shift, nb, hist);
        LS_LAUNCH_CHECK();
        k_scan_chunks<<<(unsigned)chunks, kSortThreads, 0, st>>>(hist, len, totals);
        LS_LAUNCH_CHECK();
        k_scan_totals<<<1, kSortThreads, 0, st>>>(totals, chunks);
        LS_LAUNCH_CHECK();
        k_scan_add<<<grid_for(len, 256), 256, 0, st>>>(hist, len, totals);
        LS_LAUNCH_CHECK();
        k_radix_scatter<K><<<(unsigned)nb, kSortThreads, 0, st>>>(
            kbuf[cur], vin, n, shift, nb, hist, kbuf[cur ^ 1], vbuf[cur ^ 1]);
        LS_LAUNCH_CHECK();
        vin = vbuf[cur ^ 1];  // the next pass reads what this one wrote
        cur ^= 1;
    }
    keys_res = kbuf[cur];
    vals_res = vbuf[cur];
    return 0;
}

__global__ void k_u32_to_i64(const uint32_t *__restrict__ a, int64_t n, int64_t *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        out[k] = (int64_t)a[k];
}

__global__ void k_assign(const float *__restrict__ pos, int64_t n, double ox, double oy,
                         double oz, double cell, int64_t dx, int64_t dy, int64_t dz,
                         int64_t *__restrict__ ids, uint32_t *__restrict__ keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix = __double2ll_rd(ddiv(dsub((double)pos[3 * k], ox), cell));
        int64_t iy = __double2ll_rd(ddiv(dsub((double)pos[3 * k + 1], oy), cell));
        int64_t iz = __double2ll_rd(ddiv(dsub((double)pos[3 * k + 2], oz), cell));
        ix = ix < 0 ? 0 : (ix > dx - 1 ? dx - 1 : ix);
        iy = iy < 0 ? 0 : (iy > dy - 1 ? dy - 1 : iy);
        iz = iz < 0 ? 0 : (iz > dz - 1 ? dz - 1 : iz);
        const int64_t id = (ix * dy + iy) * dz + iz;
        if (ids) ids[k] = id;
        if (keys) keys[k] = (uint32_t)id;
    }
}

__global__ void k_ids_to_keys(const int64_t *__restrict__ ids, int64_t n,
                              uint32_t *__restrict__ keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        keys[k] = (uint32_t)ids[k];
}

// offsets[c] = #keys < c  (lower bound in the sorted keys), c = 0..n_cells
__global__ void k_offsets_from_sorted(const uint32_t *__restrict__ sorted, int64_t n,
                                      int64_t n_cells, int64_t *__restrict__ offsets) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n_cells;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)sorted[mid] < c) lo = mid + 1; else hi = mid;
        }
        offsets[c] = lo;
    }
}

__global__ void k_gather(const float *__restrict__ pos, const uint8_t *__restrict__ col,
                         const int64_t *__restrict__ order, int64_t n, float *__restrict__ spos,
                         uint8_t *__restrict__ scol) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = order[k];
        spos[3 * k] = pos[3 * i];
        spos[3 * k + 1] = pos[3 * i + 1];
        spos[3 * k + 2] = pos[3 * i + 2];
        scol[3 * k] = col[3 * i];
        scol[3 * k + 1] = col[3 * i + 1];
        scol[3 * k + 2] = col[3 * i + 2];
    }
}

// Device-scan order (internal; the public grid keeps the reference's stable
// order): cell-major as before, and inside a cell by the 30-bit Morton code of
// the point's in-cell position, so consecutive points -- one warp tile -- are
// spatial neighbours that land on the same or adjacent pixels (the frame
// passes then merge same-pixel updates inside the warp).  Any in-cell order
// renders the same frame: both frame reductions are order-free.
__device__ __forceinline__ uint64_t spread3(uint32_t v) {  // 10 bits -> every 3rd of 30
    uint64_t x = v & 1023u;
    x = (x | (x << 16)) & 0x030000FFull;
    x = (x | (x << 8)) & 0x0300F00Full;
    x = (x | (x << 4)) & 0x030C30C3ull;
    x = (x | (x << 2)) & 0x09249249ull;
    return x;
}

__global__ void k_morton_keys(const float *__restrict__ pos, int64_t n, double ox, double oy,
                              double oz, double cell, int64_t dx, int64_t dy, int64_t dz,
                              uint64_t *__restrict__ keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double fx = ddiv(dsub((double)pos[3 * k], ox), cell);
        const double fy = ddiv(dsub((double)pos[3 * k + 1], oy), cell);
        const double fz = ddiv(dsub((double)pos[3 * k + 2], oz), cell);
        int64_t ix = __double2ll_rd(fx), iy = __double2ll_rd(fy), iz = __double2ll_rd(fz);
        // in-cell coordinate quantised to 10 bits (clamped: points on the far
        // faces of boundary cells)
        auto q = [](double f, int64_t i) -> uint32_t {
            const double t = (f - (double)i) * 1024.0;
            return t <= 0.0 ? 0u : (t >= 1023.0 ? 1023u : (uint32_t)t);
        };
        const uint32_t qx = q(fx, ix), qy = q(fy, iy), qz = q(fz, iz);
        ix = ix < 0 ? 0 : (ix > dx - 1 ? dx - 1 : ix);
        iy = iy < 0 ? 0 : (iy > dy - 1 ? dy - 1 : iy);
        iz = iz < 0 ? 0 : (iz > dz - 1 ? dz - 1 : iz);
        const uint64_t id = (uint64_t)((ix * dy + iy) * dz + iz);
        keys[k] = (id << 30) | spread3(qx) | (spread3(qy) << 1) | (spread3(qz) << 2);
    }
}

inline int end_bit_for(int64_t n_cells) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) < n_cells) ++b;
    return b;
}

}  // namespace ls

using namespace ls;

extern "C" {

int ls_assign_cells(const float *d_positions, int64_t n, const double origin[3], double cell_size,
                    const int64_t dims[3], int64_t *d_ids, void *stream) {
    if (n < 0 || cell_size <= 0 || !origin || !dims) return LS_EINVAL;
    if (n == 0) return 0;
    k_assign<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        d_positions, n, origin[0], origin[1], origin[2], cell_size, dims[0], dims[1], dims[2],
        d_ids, nullptr);
    LS_LAUNCH_CHECK();
    return 0;
}

size_t ls_counting_sort_workspace(int64_t n, int64_t n_cells) {
    if (n <= 0 || n_cells <= 0 || n >= (int64_t(1) << 31) || n_cells > (int64_t(1) << 32))
        return 0;
    // keys x2 (u32), values x2 (u32), sort scratch
    return a256(4 * (size_t)n) * 4 + a256(radix_scratch_bytes(n));
}

int ls_counting_sort(const int64_t *d_ids, int64_t n, int64_t n_cells, int64_t *d_offsets,
                     int64_t *d_order, void *d_workspace, size_t workspace_bytes, void *stream) {
    if (n <= 0 || n_cells <= 0) return LS_EINVAL;
    const size_t need = ls_counting_sort_workspace(n, n_cells);
    if (need == 0 || workspace_bytes < need) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)d_workspace;
    uint32_t *ka = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    uint32_t *kb = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    uint32_t *va = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    uint32_t *vb = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    k_ids_to_keys<<<grid_for(n, 256), 256, 0, st>>>(d_ids, n, ka);
    LS_LAUNCH_CHECK();
    uint32_t *keys = nullptr, *vals = nullptr;
    int rc = radix_sort<uint32_t>(ka, kb, va, vb, n, end_bit_for(n_cells), w, st, keys, vals);
    if (rc) return rc;
    k_u32_to_i64<<<grid_for(n, 256), 256, 0, st>>>(vals, n, d_order);
    LS_LAUNCH_CHECK();
    k_offsets_from_sorted<<<grid_for(n_cells + 1, 256), 256, 0, st>>>(keys, n, n_cells,
                                                                     d_offsets);
    LS_LAUNCH_CHECK();
    return 0;
}

size_t ls_morton_order_workspace(int64_t n, int64_t n_cells) {
    if (n <= 0 || n_cells <= 0 || n >= (int64_t(1) << 31) || n_cells > (int64_t(1) << 32))
        return 0;
    // keys x2 (u64), values x2 (u32), sort scratch
    return a256(8 * (size_t)n) * 2 + a256(4 * (size_t)n) * 2 + a256(radix_scratch_bytes(n));
}

int ls_morton_order(const float *d_positions, int64_t n, const double origin[3],
                    double cell_size, const int64_t dims[3], int64_t *d_order, void *d_workspace,
                    size_t workspace_bytes, void *stream) {
    if (n <= 0 || cell_size <= 0 || !origin || !dims || !d_order) return LS_EINVAL;
    const int64_t n_cells = dims[0] * dims[1] * dims[2];
    const size_t need = ls_morton_order_workspace(n, n_cells);
    if (need == 0 || workspace_bytes < need) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)d_workspace;
    uint64_t *ka = (uint64_t *)w;
    w += a256(8 * (size_t)n);
    uint64_t *kb = (uint64_t *)w;
    w += a256(8 * (size_t)n);
    uint32_t *va = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    uint32_t *vb = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    k_morton_keys<<<grid_for(n, 256), 256, 0, st>>>(d_positions, n, origin[0], origin[1],
                                                    origin[2], cell_size, dims[0], dims[1],
                                                    dims[2], ka);
    LS_LAUNCH_CHECK();
    uint64_t *keys = nullptr;
    uint32_t *vals = nullptr;
    int rc = radix_sort<uint64_t>(ka, kb, va, vb, n, 30 + end_bit_for(n_cells), w, st, keys, vals);
    if (rc) return rc;
    k_u32_to_i64<<<grid_for(n, 256), 256, 0, st>>>(vals, n, d_order);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_gather_points(const float *d_positions, const uint8_t *d_colors, const int64_t *d_order,
                     int64_t n, float *d_sorted_positions, uint8_t *d_sorted_colors,
                     void *stream) {
    if (n < 0) return LS_EINVAL;
    if (n == 0) return 0;
    k_gather<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        d_positions, d_colors, d_order, n, d_sorted_positions, d_sorted_colors);
    LS_LAUNCH_CHECK();
    return 0;
}

int ls_version(void) { return 1; }

const char *ls_status_string(int status) {
    if (status == 0) return "ok";
    if (status == LS_EINVAL) return "invalid argument";
    return cudaGetErrorString((cudaError_t)status);
}

}  // extern "C"
