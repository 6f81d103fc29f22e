// Frustum culling of occupied grid cells (grid.py:131-151) and the ordered
// warp-ballot stream compaction used for cull_cells / occupied_cells.
//
// One thread per occupied cell evaluates the CULL_SLACK-inflated p-vertex test
// in the reference's f64 operation order; a warp ballot packs 32 verdicts into
// one u32 word, which is all the frame passes need (a tile's status is a
// popcount over its cells' bits).  The drop-in cull_cells() return value
// (ascending kept ids) comes from a three-launch ordered compaction: per-block
// popcounts -> exclusive scan -> ballot-rank scatter.
#include "ls_common.cuh"

namespace ls {

struct Planes {
    double p[24];
};

__global__ void __launch_bounds__(256) k_cull(const int64_t *__restrict__ cells, int64_t n_occ,
                                              double ox, double oy, double oz, double cell,
                                              int64_t dy, int64_t dz, Planes pl, double slack,
                                              uint32_t *__restrict__ bits) {
    pdl_wait();  // the previous frame's kernels may still be draining
    const int lane = threadIdx.x & 31;
    const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = wg * 32; base < n_occ; base += nw * 32) {
        const int64_t j = base + lane;
        bool keep = false;
        if (j < n_occ) {
            const int64_t c = cells[j];
            const int64_t iz = c % dz, iy = (c / dz) % dy, ix = c / (dy * dz);
            // cell_boxes (grid.py:69-76): lo = origin + idx*cell, hi = lo + cell
            const double o[3] = {ox, oy, oz};
            const double idx[3] = {(double)ix, (double)iy, (double)iz};
            double lo[3], hi[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double l = dadd(o[a], dmul(idx[a], cell));
                hi[a] = dadd(dadd(l, cell), slack);
                lo[a] = dsub(l, slack);
            }
            keep = true;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const double nx = pl.p[4 * q], ny = pl.p[4 * q + 1], nz = pl.p[4 * q + 2],
                             d = pl.p[4 * q + 3];
                const double px = nx >= 0 ? hi[0] : lo[0];
                const double py = ny >= 0 ? hi[1] : lo[1];
                const double pz = nz >= 0 ? hi[2] : lo[2];
                const double s = dadd(dadd(dadd(dmul(px, nx), dmul(py, ny)), dmul(pz, nz)), d);
                keep = keep && (s >= 0.0);
            }
        }
        const uint32_t word = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) bits[base >> 5] = word;
    }
    pdl_trigger();
}

// predicate bits for occupied cells: offsets[c+1] > offsets[c]
__global__ void k_occupied_bits(const int64_t *__restrict__ off, int64_t n_cells,
                                uint32_t *__restrict__ bits) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = wg * 32; base < n_cells; base += nw * 32) {
        const int64_t c = base + lane;
        const bool occ = c < n_cells && off[c + 1] > off[c];
        const uint32_t word = __ballot_sync(0xffffffffu, occ);
        if (lane == 0) bits[base >> 5] = word;
    }
}

constexpr int kCompactBlock = 1024;  // 32 words = 1024 items per CTA

__global__ void k_block_popc(const uint32_t *__restrict__ bits, int64_t n_words,
                             int64_t *__restrict__ counts) {
    __shared__ int64_t part[32];
    const int64_t w = blockIdx.x * 32ll + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    int c = 0;
    if (lane == 0 && w < n_words) c = __popc(bits[w]);
    if (lane == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = part[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) counts[blockIdx.x] = v;
    }
}

// single-CTA exclusive scan with a serial carry; writes total to *total and,
// if tail_dst != nullptr, tail_dst[total] = tail_val
__global__ void k_scan_exclusive(const int64_t *__restrict__ in, int64_t n,
                                 int64_t *__restrict__ out, int64_t *__restrict__ total,
                                 int64_t *__restrict__ tail_dst, const int64_t *__restrict__ tail_src) {
    __shared__ int64_t carry;
    __shared__ int64_t wt[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int64_t x = i < n ? in[i] : 0;
        int64_t v = x;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) wt[wid] = v;
        __syncthreads();
        if (wid == 0) {
            int64_t t = lane < (int)(blockDim.x >> 5) ? wt[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int64_t u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            wt[lane] = t;
        }
        __syncthreads();
        const int64_t incl = v + (wid > 0 ? wt[wid - 1] : 0) + carry;
        if (i < n) out[i] = incl - x;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *total = carry;
        if (tail_dst) tail_dst[carry] = *tail_src;
    }
}

// scatter: item j with its bit set goes to out position block_off + rank
template <bool OCCUPIED>
__global__ void k_compact_scatter(const uint32_t *__restrict__ bits, int64_t n_words,
                                  const int64_t *__restrict__ block_off,
                                  const int64_t *__restrict__ src, int64_t *__restrict__ out_a,
                                  int64_t *__restrict__ out_b) {
    __shared__ int wpre[32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * 32ll + wid;
    const uint32_t word = w < n_words ? bits[w] : 0u;
    if (lane == 0) wpre[wid] = __popc(word);
    __syncthreads();
    if (threadIdx.x < 32) {
        int v = wpre[threadIdx.x], incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        wpre[threadIdx.x] = incl - v;
    }
    __syncthreads();
    if ((word >> lane) & 1u) {
        const int64_t pos = block_off[blockIdx.x] + wpre[wid] + __popc(word & ((1u << lane) - 1u));
        const int64_t j = w * 32 + lane;
        if (OCCUPIED) {
            out_a[pos] = j;         // cell id
            out_b[pos] = src[j];    // its point offset
        } else {
            out_a[pos] = src[j];    // kept occupied cell id
        }
    }
}

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace ls

namespace ls {
// (for ls_frame_graph_set_camera: the captured node to re-target, and the
// index of its Planes argument)
const void *cull_kernel() { return (const void *)k_cull; }
constexpr int kCullPlanesArg = 8;
int cull_planes_arg() { return kCullPlanesArg; }
}  // namespace ls

using namespace ls;

extern "C" {

int ls_cull(const ls_scene *scene, const double h_planes[24], double slack,
            uint32_t *d_keep_bits, void *stream) {
    if (!scene || !h_planes || !d_keep_bits || scene->n_occ < 0 || scene->cell_size <= 0)
        return LS_EINVAL;
    if (scene->n_occ == 0) return 0;
    Planes pl;
    for (int i = 0; i < 24; ++i) pl.p[i] = h_planes[i];
    const int64_t n_words = (scene->n_occ + 31) / 32;
    cudaError_t e = launch_pdl(k_cull, dim3(grid_for(n_words * 32, 256)), dim3(256), 0,
                               (cudaStream_t)stream, scene->d_occ_cells, scene->n_occ,
                               scene->origin[0], scene->origin[1], scene->origin[2],
                               scene->cell_size, scene->dims[1], scene->dims[2], pl, slack,
                               d_keep_bits);
    return (int)e;
}

size_t ls_compact_workspace(int64_t n_items) {
    const int64_t nb = (n_items + kCompactBlock - 1) / kCompactBlock;
    return align256(sizeof(int64_t) * (size_t)(nb + 1)) * 2;
}

int ls_cull_compact(const uint32_t *d_keep_bits, const int64_t *d_occ_cells, int64_t n_occ,
                    int64_t *d_out_cells, int64_t *d_count, void *d_workspace,
                    size_t workspace_bytes, void *stream) {
    if (n_occ < 0 || workspace_bytes < ls_compact_workspace(n_occ)) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_occ == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(int64_t), st);
        return e == cudaSuccess ? 0 : (int)e;
    }
    const int64_t nb = (n_occ + kCompactBlock - 1) / kCompactBlock;
    const int64_t n_words = (n_occ + 31) / 32;
    int64_t *counts = (int64_t *)d_workspace;
    int64_t *offs = (int64_t *)((char *)d_workspace + align256(sizeof(int64_t) * (nb + 1)));
    k_block_popc<<<(unsigned)nb, kCompactBlock, 0, st>>>(d_keep_bits, n_words, counts);
    LS_LAUNCH_CHECK();
    k_scan_exclusive<<<1, 1024, 0, st>>>(counts, nb, offs, d_count, nullptr, nullptr);
    LS_LAUNCH_CHECK();
    k_compact_scatter<false><<<(unsigned)nb, kCompactBlock, 0, st>>>(
        d_keep_bits, n_words, offs, d_occ_cells, d_out_cells, nullptr);
    LS_LAUNCH_CHECK();
    return 0;
}

size_t ls_occupied_workspace(int64_t n_cells) {
    const int64_t n_words = (n_cells + 31) / 32;
    return align256(sizeof(uint32_t) * (size_t)n_words) + ls_compact_workspace(n_cells);
}

int ls_occupied_cells(const int64_t *d_cell_offsets, int64_t n_cells, int64_t *d_occ_cells,
                      int64_t *d_occ_offsets, int64_t *d_n_occ, void *d_workspace,
                      size_t workspace_bytes, void *stream) {
    if (n_cells <= 0 || workspace_bytes < ls_occupied_workspace(n_cells)) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n_words = (n_cells + 31) / 32;
    const int64_t nb = (n_cells + kCompactBlock - 1) / kCompactBlock;
    uint32_t *bits = (uint32_t *)d_workspace;
    char *rest = (char *)d_workspace + align256(sizeof(uint32_t) * n_words);
    int64_t *counts = (int64_t *)rest;
    int64_t *offs = (int64_t *)(rest + align256(sizeof(int64_t) * (nb + 1)));
    k_occupied_bits<<<grid_for(n_words * 32, 256), 256, 0, st>>>(d_cell_offsets, n_cells, bits);
    LS_LAUNCH_CHECK();
    k_block_popc<<<(unsigned)nb, kCompactBlock, 0, st>>>(bits, n_words, counts);
    LS_LAUNCH_CHECK();
    // occ_offsets[n_occ] = cell_offsets[n_cells] (= n_points)
    k_scan_exclusive<<<1, 1024, 0, st>>>(counts, nb, offs, d_n_occ, d_occ_offsets,
                                         d_cell_offsets + n_cells);
    LS_LAUNCH_CHECK();
    k_compact_scatter<true><<<(unsigned)nb, kCompactBlock, 0, st>>>(
        bits, n_words, offs, d_cell_offsets, d_occ_cells, d_occ_offsets);
    LS_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
