// Per-scan grid build on the device (grid.py:94-128): cell assignment, the
// stable counting sort and the cell-major gathers.
//
// assign_cells is a bit-exact f64 restatement of _native.pyx:19-44.  The stable
// sort is an LSD radix sort of u32 cell ids carrying the i64 point index (CUB,
// the CUDA toolkit's header-only device library; radix sort is stable, so the
// permutation equals the reference's counting sort / argsort(kind="stable")),
// followed by a lower-bound pass that materialises cell_offsets.
#include <cub/device/device_radix_sort.cuh>

#include "ls_common.cuh"

namespace ls {

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
                              uint32_t *__restrict__ keys, int64_t *__restrict__ iota) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        keys[k] = (uint32_t)ids[k];
        iota[k] = k;
    }
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
                              uint64_t *__restrict__ keys, int64_t *__restrict__ iota) {
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
        iota[k] = k;
    }
}

inline int end_bit_for(int64_t n_cells) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) < n_cells) ++b;
    return b;
}

inline size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

size_t cub_temp_bytes(int64_t n, int64_t n_cells) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, (int)n, 0,
                                    end_bit_for(n_cells));
    return temp;
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
    return a256(4 * (size_t)n) * 2 + a256(8 * (size_t)n) + a256(cub_temp_bytes(n, n_cells));
}

int ls_counting_sort(const int64_t *d_ids, int64_t n, int64_t n_cells, int64_t *d_offsets,
                     int64_t *d_order, void *d_workspace, size_t workspace_bytes, void *stream) {
    if (n <= 0 || n_cells <= 0) return LS_EINVAL;
    const size_t need = ls_counting_sort_workspace(n, n_cells);
    if (need == 0 || workspace_bytes < need) return LS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)d_workspace;
    uint32_t *keys_in = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    uint32_t *keys_out = (uint32_t *)w;
    w += a256(4 * (size_t)n);
    int64_t *iota = (int64_t *)w;
    w += a256(8 * (size_t)n);
    size_t temp = cub_temp_bytes(n, n_cells);
    k_ids_to_keys<<<grid_for(n, 256), 256, 0, st>>>(d_ids, n, keys_in, iota);
    LS_LAUNCH_CHECK();
    cudaError_t e = cub::DeviceRadixSort::SortPairs(w, temp, keys_in, keys_out, iota, d_order,
                                                    (int)n, 0, end_bit_for(n_cells), st);
    if (e != cudaSuccess) return (int)e;
    k_offsets_from_sorted<<<grid_for(n_cells + 1, 256), 256, 0, st>>>(keys_out, n, n_cells,
                                                                     d_offsets);
    LS_LAUNCH_CHECK();
    return 0;
}

size_t ls_morton_order_workspace(int64_t n, int64_t n_cells) {
    if (n <= 0 || n_cells <= 0 || n >= (int64_t(1) << 31) || n_cells > (int64_t(1) << 32))
        return 0;
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, (int)n, 0,
                                    30 + end_bit_for(n_cells));
    return a256(8 * (size_t)n) * 3 + a256(temp);
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
    uint64_t *keys_in = (uint64_t *)w;
    w += a256(8 * (size_t)n);
    uint64_t *keys_out = (uint64_t *)w;
    w += a256(8 * (size_t)n);
    int64_t *iota = (int64_t *)w;
    w += a256(8 * (size_t)n);
    size_t temp = need - 3 * a256(8 * (size_t)n);
    k_morton_keys<<<grid_for(n, 256), 256, 0, st>>>(d_positions, n, origin[0], origin[1],
                                                    origin[2], cell_size, dims[0], dims[1],
                                                    dims[2], keys_in, iota);
    LS_LAUNCH_CHECK();
    cudaError_t e = cub::DeviceRadixSort::SortPairs(w, temp, keys_in, keys_out, iota, d_order,
                                                    (int)n, 0, 30 + end_bit_for(n_cells), st);
    return (int)e;
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
