/*
 * oracle_kernels.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference's per-frame hot loops
 * (arxiv 2502.11618 "lidarsplat", /root/reference/pkg/src/lidarsplat/_kernels).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2502_11618_b200/) never links or imports it.
 *
 * Arithmetic contract (reference _kernels/_numpy.py:3-13): positions widened
 * to f64, left-associated products, one rounding per op (built with
 * -ffp-contract=off exactly like pkg/setup.py:13-15), u64 colour sums.
 *
 * Pinned against the reference's own known-answer tests and against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef uint64_t u64;
typedef uint8_t u8;

static i64 clamp_i64(i64 v, i64 lo, i64 hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* reference: _native.pyx:19-44 (assign_cells), _numpy.py:20-25 */
void or_assign_cells(const float *pos, i64 n, const double *origin, double cell,
                     const i64 *dims, i64 *ids) {
    for (i64 k = 0; k < n; ++k) {
        i64 ix = (i64)floor(((double)pos[3 * k + 0] - origin[0]) / cell);
        i64 iy = (i64)floor(((double)pos[3 * k + 1] - origin[1]) / cell);
        i64 iz = (i64)floor(((double)pos[3 * k + 2] - origin[2]) / cell);
        ix = clamp_i64(ix, 0, dims[0] - 1);
        iy = clamp_i64(iy, 0, dims[1] - 1);
        iz = clamp_i64(iz, 0, dims[2] - 1);
        ids[k] = (ix * dims[1] + iy) * dims[2] + iz;
    }
}

/* reference: _native.pyx:47-68 (stable counting sort) */
int or_counting_sort(const i64 *ids, i64 n, i64 n_cells, i64 *offsets, i64 *order) {
    i64 *cursor = (i64 *)malloc(sizeof(i64) * (size_t)(n_cells > 0 ? n_cells : 1));
    if (!cursor) return -1;
    memset(offsets, 0, sizeof(i64) * (size_t)(n_cells + 1));
    for (i64 k = 0; k < n; ++k) offsets[ids[k] + 1] += 1;
    for (i64 c = 0; c < n_cells; ++c) {
        offsets[c + 1] += offsets[c];
        cursor[c] = offsets[c];
    }
    for (i64 k = 0; k < n; ++k) order[cursor[ids[k]]++] = k;
    free(cursor);
    return 0;
}

/* Camera transform + clip + pixel of one point.  Returns the pixel index, or
 * -1 when the point does not rasterize; *zc_out always receives the camera z.
 * reference: _native.pyx:98-117, _numpy.py:47-66 */
static i64 project_one(const float *p, const double *r, const double *t, double fx,
                       double fy, double cx, double cy, i64 w, i64 h, double zn,
                       double zf, double *zc_out) {
    double x = (double)p[0], y = (double)p[1], z = (double)p[2];
    double zc = (r[6] * x + r[7] * y) + r[8] * z + t[2];
    *zc_out = zc;
    if (!(zc >= zn && zc <= zf)) return -1; /* NaN never rasterizes (numpy rule) */
    double xc = (r[0] * x + r[1] * y) + r[2] * z + t[0];
    double yc = (r[3] * x + r[4] * y) + r[5] * z + t[1];
    double invz = 1.0 / zc;
    double u = (fx * xc) * invz + cx;
    if (!(u >= 0.0 && u < (double)w)) return -1;
    double v = (fy * yc) * invz + cy;
    if (!(v >= 0.0 && v < (double)h)) return -1;
    return (i64)floor(v) * w + (i64)floor(u);
}

/* Pass 1. reference: _native.pyx:71-121 */
void or_project_min_depth(const float *pos, const i64 *starts, const i64 *ends, i64 nr,
                          const double *rot, const double *t, double fx, double fy,
                          double cx, double cy, i64 w, i64 h, double zn, double zf,
                          double *minz, i64 *pix_cache, double *z_cache) {
    i64 k = 0;
    for (i64 r = 0; r < nr; ++r) {
        for (i64 i = starts[r]; i < ends[r]; ++i, ++k) {
            double zc;
            i64 pix = project_one(pos + 3 * i, rot, t, fx, fy, cx, cy, w, h, zn, zf, &zc);
            z_cache[k] = zc;
            pix_cache[k] = pix;
            if (pix >= 0 && zc < minz[pix]) minz[pix] = zc;
        }
    }
}

/* Pass 2. reference: _native.pyx:124-148 */
void or_project_accumulate(const u8 *col, const i64 *starts, const i64 *ends, i64 nr,
                           const i64 *pix_cache, const double *z_cache, double eps_rel,
                           const double *minz, u64 *accum) {
    const double one_plus_eps = 1.0 + eps_rel;
    i64 k = 0;
    for (i64 r = 0; r < nr; ++r) {
        for (i64 i = starts[r]; i < ends[r]; ++i, ++k) {
            i64 pix = pix_cache[k];
            if (pix < 0) continue;
            if (z_cache[k] <= minz[pix] * one_plus_eps) {
                u64 *a = accum + 4 * pix;
                a[0] += col[3 * i + 0];
                a[1] += col[3 * i + 1];
                a[2] += col[3 * i + 2];
                a[3] += 1;
            }
        }
    }
}

/* Frame assembly. reference: render.py:146-161 (assemble_frame) */
void or_assemble(const double *minz, const u64 *accum, i64 npix, float *rgb, float *depth,
                 u8 *alpha) {
    for (i64 p = 0; p < npix; ++p) {
        const u64 *a = accum + 4 * p;
        if (a[3] > 0) {
            double denom = (double)a[3] * 255.0;
            rgb[3 * p + 0] = (float)((double)a[0] / denom);
            rgb[3 * p + 1] = (float)((double)a[1] / denom);
            rgb[3 * p + 2] = (float)((double)a[2] / denom);
            depth[p] = (float)minz[p];
            alpha[p] = 1;
        } else {
            rgb[3 * p + 0] = rgb[3 * p + 1] = rgb[3 * p + 2] = 0.0f;
            depth[p] = 0.0f;
            alpha[p] = 0;
        }
    }
}

/* reference: _native.pyx:151-170 (ceil-size 2x2 min pool, missing children skipped) */
void or_min_pool_2x2(const float *img, i64 h, i64 w, float *out) {
    i64 oh = (h + 1) / 2, ow = (w + 1) / 2;
    for (i64 y = 0; y < oh; ++y) {
        for (i64 x = 0; x < ow; ++x) {
            float m = INFINITY;
            for (i64 dy = 0; dy < 2; ++dy) {
                i64 sy = 2 * y + dy;
                if (sy >= h) break;
                for (i64 dx = 0; dx < 2; ++dx) {
                    i64 sx = 2 * x + dx;
                    if (sx >= w) break;
                    float v = img[sy * w + sx];
                    if (v < m) m = v;
                }
            }
            out[y * ow + x] = m;
        }
    }
}

/* reference: _native.pyx:173-196 */
void or_laplacian_edges(const float *img, i64 h, i64 w, double thr, u8 *out) {
    for (i64 y = 0; y < h; ++y) {
        for (i64 x = 0; x < w; ++x) {
            double c = (double)img[y * w + x];
            out[y * w + x] = 0;
            if (!isfinite(c)) continue;
            double nb[4] = {y > 0 ? (double)img[(y - 1) * w + x] : c,
                            y + 1 < h ? (double)img[(y + 1) * w + x] : c,
                            x > 0 ? (double)img[y * w + x - 1] : c,
                            x + 1 < w ? (double)img[y * w + x + 1] : c};
            for (int j = 0; j < 4; ++j)
                if (!isfinite(nb[j])) nb[j] = c;
            double resp = (((nb[0] + nb[1]) + nb[2]) + nb[3]) - 4.0 * c;
            if (fabs(resp) > thr * c) out[y * w + x] = 1;
        }
    }
}

/* reference: _native.pyx:199-237 (max-rule reference; equivalent to the
 * existential rule of tests/reference.py:116-172) */
void or_filter_keep(const float *coarse, i64 ch, i64 cw, const u8 *edges, const float *fine,
                    i64 fh, i64 fw, double fs, float *out) {
    for (i64 i = 0; i < fh * fw; ++i) out[i] = INFINITY;
    for (i64 cy = 0; cy < ch; ++cy) {
        for (i64 cx = 0; cx < cw; ++cx) {
            double c = (double)coarse[cy * cw + cx];
            double ref = isfinite(c) ? c : -INFINITY;
            if (edges[cy * cw + cx]) {
                for (i64 ny = cy - 1; ny <= cy + 1; ++ny) {
                    if (ny < 0 || ny >= ch) continue;
                    for (i64 nx = cx - 1; nx <= cx + 1; ++nx) {
                        if (nx < 0 || nx >= cw || (ny == cy && nx == cx)) continue;
                        double v = (double)coarse[ny * cw + nx];
                        if (isfinite(v) && v > ref) ref = v;
                    }
                }
            }
            if (!isfinite(ref)) continue;
            for (i64 fy = 2 * cy; fy < 2 * cy + 2 && fy < fh; ++fy) {
                for (i64 fx = 2 * cx; fx < 2 * cx + 2 && fx < fw; ++fx) {
                    double f = (double)fine[fy * fw + fx];
                    if (isfinite(f) && (f - ref) <= fs * ref) out[fy * fw + fx] = fine[fy * fw + fx];
                }
            }
        }
    }
}

/* reference: _native.pyx:240-297 (renormalised bilinear, order 00,01,10,11) */
void or_bilinear_fill(const float *coarse, i64 ch, i64 cw, const float *fine, i64 fh, i64 fw,
                      float *out) {
    for (i64 y = 0; y < fh; ++y) {
        double gy = 0.5 * (double)y - 0.25;
        i64 y0r = (i64)floor(gy);
        double wy1 = gy - (double)y0r, wy0 = 1.0 - wy1;
        i64 ys[2] = {clamp_i64(y0r, 0, ch - 1), clamp_i64(y0r + 1, 0, ch - 1)};
        double wys[2] = {wy0, wy1};
        for (i64 x = 0; x < fw; ++x) {
            float fv = fine[y * fw + x];
            if (isfinite(fv)) {
                out[y * fw + x] = fv;
                continue;
            }
            double gx = 0.5 * (double)x - 0.25;
            i64 x0r = (i64)floor(gx);
            double wx1 = gx - (double)x0r, wx0 = 1.0 - wx1;
            i64 xs[2] = {clamp_i64(x0r, 0, cw - 1), clamp_i64(x0r + 1, 0, cw - 1)};
            double wxs[2] = {wx0, wx1};
            double num = 0.0, den = 0.0;
            for (int a = 0; a < 2; ++a) {
                for (int b = 0; b < 2; ++b) {
                    double v = (double)coarse[ys[a] * cw + xs[b]];
                    if (isfinite(v)) {
                        double wgt = wys[a] * wxs[b];
                        num = num + wgt * v;
                        den = den + wgt;
                    }
                }
            }
            out[y * fw + x] = den > 0.0 ? (float)(num / den) : INFINITY;
        }
    }
}

/* Frustum cull of occupied cells: CULL_SLACK-inflated AABB, p-vertex test.
 * reference: grid.py:131-151 (cull_cells) + grid.py:69-76 (cell_boxes).
 * keep[j] = 1 iff cell cells[j] survives all six planes. */
void or_cull_cells(const i64 *cells, i64 n, const double *origin, double cell,
                   const i64 *dims, const double *planes, double slack, u8 *keep) {
    i64 dy = dims[1], dz = dims[2];
    for (i64 j = 0; j < n; ++j) {
        i64 c = cells[j];
        i64 iz = c % dz, iy = (c / dz) % dy, ix = c / (dy * dz);
        double idx[3] = {(double)ix, (double)iy, (double)iz};
        double lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            double l = origin[a] + idx[a] * cell;
            hi[a] = (l + cell) + slack;
            lo[a] = l - slack;
        }
        u8 k = 1;
        for (int p = 0; p < 6; ++p) {
            const double *pl = planes + 4 * p;
            double px = pl[0] >= 0 ? hi[0] : lo[0];
            double py = pl[1] >= 0 ? hi[1] : lo[1];
            double pz = pl[2] >= 0 ? hi[2] : lo[2];
            if (!(((px * pl[0] + py * pl[1]) + pz * pl[2]) + pl[3] >= 0)) k = 0;
        }
        keep[j] = k;
    }
}
