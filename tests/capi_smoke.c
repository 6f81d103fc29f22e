/*
 * The C ABI without Python: what a C/C++ (or cgo/JNI) caller of
 * include/lidarsplat_cuda.h does for one frame.  Builds a tiny scene on the
 * device through the ABI (assign cells -> stable sort -> gather -> occupied
 * cells -> tile index), renders it with ls_frame_project + ls_frame_finish,
 * and checks the pixels the reference's rules predict: a lone point, two
 * points within the soft z-buffer tolerance (mean colour), an occluded point,
 * and a point outside the frame.  Prints "capi_smoke OK" on success.
 *
 *   gcc capi_smoke.c -I../include -L../paper_2502_11618_b200 -llidarsplat_cuda \
 *       -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o capi_smoke
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lidarsplat_cuda.h"

#define CK(x)                                                                        \
    do {                                                                             \
        int rc__ = (int)(x);                                                         \
        if (rc__) {                                                                  \
            fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc__,  \
                    ls_status_string(rc__));                                         \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static void *dalloc(size_t bytes) {
    void *p = NULL;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return NULL;
    return p;
}

int main(void) {
    enum { W = 64, H = 48, N = 5 };
    /* camera at the origin looking down +z: pixel (u, v) = (fx x/z + cx, fy y/z + cy) */
    ls_camera cam;
    memset(&cam, 0, sizeof cam);
    cam.rot[0] = cam.rot[4] = cam.rot[8] = 1.0;
    cam.fx = cam.fy = 40.0;
    cam.cx = 32.0;
    cam.cy = 24.0;
    cam.width = W;
    cam.height = H;
    cam.z_near = 0.1;
    cam.z_far = 100.0;
    /* every point projects to a pixel centre, far from pixel boundaries */
    const float pos[N][3] = {
        {0.05f, 0.05f, 4.0f},               /* lone point        -> (32.5, 24.5) */
        {-0.475f, -0.225f, 2.0f},           /* pair, front       -> (22.5, 19.5) */
        {-0.477375f, -0.226125f, 2.01f},    /* pair, within 1%   -> (22.5, 19.5) */
        {-1.425f, -0.675f, 6.0f},           /* behind the pair   -> (22.5, 19.5) */
        {40.0f, 0.0f, 4.0f},                /* outside the frame                  */
    };
    const unsigned char col[N][3] = {{200, 10, 20}, {100, 0, 50}, {0, 200, 150},
                                     {255, 255, 255}, {1, 2, 3}};
    const double origin[3] = {-2.0, -1.0, 1.0};
    const double cell = 1.0;
    const int64_t dims[3] = {43, 2, 6};
    const int64_t n_cells = dims[0] * dims[1] * dims[2];
    cudaStream_t st = 0;

    float *d_pos = dalloc(sizeof pos), *d_spos = dalloc(sizeof pos);
    unsigned char *d_col = dalloc(sizeof col), *d_scol = dalloc(sizeof col);
    int64_t *d_ids = dalloc(8 * N), *d_order = dalloc(8 * N);
    int64_t *d_offsets = dalloc(8 * (n_cells + 1));
    if (!d_pos || !d_spos || !d_col || !d_scol || !d_ids || !d_order || !d_offsets) return 2;
    cudaMemcpy(d_pos, pos, sizeof pos, cudaMemcpyHostToDevice);
    cudaMemcpy(d_col, col, sizeof col, cudaMemcpyHostToDevice);

    /* per-scan: grid build (R:grid.py:94-128) */
    CK(ls_assign_cells(d_pos, N, origin, cell, dims, d_ids, st));
    size_t ws_bytes = ls_counting_sort_workspace(N, n_cells);
    void *ws = dalloc(ws_bytes);
    CK(ls_counting_sort(d_ids, N, n_cells, d_offsets, d_order, ws, ws_bytes, st));
    CK(ls_gather_points(d_pos, d_col, d_order, N, d_spos, d_scol, st));
    /* per-scan: occupied cells + tile index */
    size_t ows = ls_occupied_workspace(n_cells);
    void *ows_p = dalloc(ows);
    int64_t *d_occ = dalloc(8 * n_cells), *d_occ_off = dalloc(8 * (n_cells + 1)),
            *d_nocc = dalloc(8);
    CK(ls_occupied_cells(d_offsets, n_cells, d_occ, d_occ_off, d_nocc, ows_p, ows, st));
    int64_t n_occ = 0;
    cudaMemcpy(&n_occ, d_nocc, 8, cudaMemcpyDeviceToHost);
    const int64_t n_tiles = (N + LS_TILE_POINTS - 1) / LS_TILE_POINTS;
    int32_t *d_c0 = dalloc(4 * n_tiles), *d_c1 = dalloc(4 * n_tiles);
    CK(ls_scene_tile_index(d_occ_off, n_occ, N, d_c0, d_c1, st));

    ls_scene sc;
    memset(&sc, 0, sizeof sc);
    sc.d_positions = d_spos;
    sc.d_colors = d_scol;
    sc.n_points = N;
    sc.d_occ_cells = d_occ;
    sc.d_occ_offsets = d_occ_off;
    sc.n_occ = n_occ;
    sc.d_tile_c0 = d_c0;
    sc.d_tile_c1 = d_c1;
    sc.n_tiles = n_tiles;
    memcpy(sc.origin, origin, sizeof origin);
    sc.cell_size = cell;
    memcpy(sc.dims, dims, sizeof dims);

    /* per frame: both passes (no cull: every point is a candidate) + assemble */
    uint64_t *d_minz = dalloc(8 * W * H);
    float *d_acc = dalloc(16 * W * H);
    uint64_t *h_inf = malloc(8 * W * H);
    for (int i = 0; i < W * H; ++i) h_inf[i] = 0x7FF0000000000000ull;
    cudaMemcpy(d_minz, h_inf, 8 * W * H, cudaMemcpyHostToDevice);
    cudaMemset(d_acc, 0, 16 * W * H);
    CK(ls_frame_project(&sc, NULL, NULL, NULL, &cam, 0.01, d_minz, NULL, d_acc, st));
    float *d_rgb = dalloc(12 * W * H), *d_depth = dalloc(4 * W * H);
    unsigned char *d_alpha = dalloc(W * H);
    int32_t *d_flags = dalloc(4);
    cudaMemset(d_flags, 0, 4);
    CK(ls_frame_finish(d_minz, d_acc, W, H, NULL, d_rgb, d_depth, d_alpha, NULL, NULL, NULL,
                       NULL, NULL, 0, 0, 0.1, NULL, d_flags, st));
    static float rgb[H][W][3], depth[H][W];
    static unsigned char alpha[H][W];
    int32_t flags = -1;
    CK(cudaMemcpy(rgb, d_rgb, sizeof rgb, cudaMemcpyDeviceToHost));
    cudaMemcpy(depth, d_depth, sizeof depth, cudaMemcpyDeviceToHost);
    cudaMemcpy(alpha, d_alpha, sizeof alpha, cudaMemcpyDeviceToHost);
    cudaMemcpy(&flags, d_flags, 4, cudaMemcpyDeviceToHost);

    int bad = 0, filled = 0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) filled += alpha[y][x];
    if (filled != 2) ++bad, fprintf(stderr, "filled pixels %d, expected 2\n", filled);
    if (flags != 0) ++bad, fprintf(stderr, "flags %d\n", flags);
    /* lone point: its colour / 255 (f64 divide, rounded to f32) and depth */
    if (!alpha[24][32] || depth[24][32] != 4.0f || rgb[24][32][0] != (float)(200.0 / 255.0) ||
        rgb[24][32][1] != (float)(10.0 / 255.0) || rgb[24][32][2] != (float)(20.0 / 255.0))
        ++bad, fprintf(stderr, "lone point wrong\n");
    /* pair within 1%: mean of both colours; the point behind is excluded */
    const double d2 = 2.0 * 255.0;
    if (!alpha[19][22] || depth[19][22] != 2.0f || rgb[19][22][0] != (float)(100.0 / d2) ||
        rgb[19][22][1] != (float)(200.0 / d2) || rgb[19][22][2] != (float)(200.0 / d2))
        ++bad, fprintf(stderr, "soft z-buffer pair wrong: %g %g %g depth %g\n", rgb[19][22][0],
                       rgb[19][22][1], rgb[19][22][2], depth[19][22]);
    if (bad) return 3;
    printf("capi_smoke OK (ls_version %d)\n", ls_version());
    return 0;
}
